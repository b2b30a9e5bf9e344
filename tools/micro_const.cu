// Microbenchmark: FP64 outer-product contraction with the operator in __constant__ memory (LDCU -> UR
// operand) vs shared memory (LDS broadcast), thread per element, NP x NP table, R elements per thread.
// Reports achieved FP64 TF/s vs resident warps.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NP = 15;
__constant__ double ctab[2 * NP * NP];

template <int R, bool SMEM>
__global__ void kern(const double* __restrict__ in, double* __restrict__ out, int reps, int zero) {
  __shared__ double stab[2 * NP * NP];
  if (SMEM) {
    for (int i = threadIdx.x; i < 2 * NP * NP; i += blockDim.x) stab[i] = ctab[i];
    __syncthreads();
  }
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  double u[R][NP];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < NP; ++j) u[r][j] = in[(t * R + r) * NP + j];
  for (int it = 0; it < reps; ++it) {
    const double* T = (SMEM ? stab : ctab) + it * zero;  // runtime 0: the loads cannot be hoisted
    double a[R][NP], b[R][NP];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int i = 0; i < NP; ++i) a[r][i] = b[r][i] = 0.0;
#pragma unroll
    for (int j = 0; j < NP; ++j)
#pragma unroll
      for (int i = 0; i < NP; ++i)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          a[r][i] = fma(T[j * NP + i], u[r][j], a[r][i]);
          b[r][i] = fma(T[NP * NP + j * NP + i], u[r][j], b[r][i]);
        }
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int i = 0; i < NP; ++i) u[r][i] = a[r][i] * 0.5 + b[r][i] * 0.25;
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < NP; ++j) out[(t * R + r) * NP + j] = u[r][j];
}

template <int R, bool SMEM>
void run(int tpb, int bpsm, int sms) {
  const int blocks = bpsm * sms, n = blocks * tpb * R, reps = 200;
  double *in, *out;
  cudaMalloc(&in, n * NP * 8);
  cudaMalloc(&out, n * NP * 8);
  cudaMemset(in, 0, n * NP * 8);
  kern<R, SMEM><<<blocks, tpb>>>(in, out, 2, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<R, SMEM><<<blocks, tpb>>>(in, out, reps, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flop = 2.0 * 2 * NP * NP * (double)n * reps;
  printf("{\"R\": %d, \"smem\": %d, \"warps_per_sm\": %d, \"tflops\": %.2f}\n", R, (int)SMEM, bpsm * tpb / 32, flop / ms / 1e9);
  cudaFree(in);
  cudaFree(out);
}

int main() {
  double h[2 * NP * NP];
  for (int i = 0; i < 2 * NP * NP; ++i) h[i] = 1e-3 * (i % 17);
  cudaMemcpyToSymbol(ctab, h, sizeof(h));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 12, 16, 24, 32}) {
    run<1, false>(128, w / 4, sms);
    run<1, true>(128, w / 4, sms);
    run<2, false>(128, w / 4, sms);
    run<2, true>(128, w / 4, sms);
  }
  return 0;
}
