// DMMA / DFMA latency and per-warp throughput on one SM (1 CTA, 1..32 warps), chain lengths 1..8.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double* out, long long* cyc, int iters) {
  double c[CH][2];
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = threadIdx.x;
  const double a = 1.0000001, b = 0.999999;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int CH>
void run(int warps) {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8);
  const int iters = 2000;
  k<CH><<<1, 32 * warps>>>(o, c, iters);
  cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("{\"chains_per_warp\": %d, \"warps\": %d, \"cycles_per_dmma_per_warp\": %.2f, \"sm_cycles_per_dmma\": %.2f}\n", CH, warps,
         (double)h / (iters * CH), (double)h / (iters * CH * warps));
  cudaFree(o); cudaFree(c);
}
int main() {
  for (int w : {1, 4, 8, 16, 32}) { run<1>(w); run<2>(w); run<4>(w); run<8>(w); }
  return 0;
}
