// Microbenchmarks for the FP64 roofline denominators on B200 (sm_100a):
// DFMA register peak, DFMA fed by shared-memory broadcast, DFMA with
// constant-bank operands, DMMA (mma.sync f64) peak for the shapes sm_100a
// accepts, DFMA+DMMA co-issue, and a device copy bandwidth.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_fp64 micro_fp64.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int ITERS = 4096;

__global__ void k_dfma(double* out, double a, double b) {
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

// one LDS.128 broadcast feeds 2 x (NE) DFMA: NE independent "elements" per thread
template <int NE>
__global__ void k_dfma_lds(double* out, const double* gop) {
  __shared__ double2 op[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) op[i] = make_double2(gop[2 * i], gop[2 * i + 1]);
  __syncthreads();
  double acc[NE], x[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) { acc[e] = 0; x[e] = threadIdx.x * 1e-3 + e; }
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      double2 d = op[(it + j) & 255];
#pragma unroll
      for (int e = 0; e < NE; ++e) { acc[e] = fma(d.x, x[e], acc[e]); x[e] = fma(d.y, acc[e], x[e]); }
    }
  }
  double s = 0;
#pragma unroll
  for (int e = 0; e < NE; ++e) s += acc[e] + x[e];
  if (s == 12345.678) out[0] = s;
}

__constant__ double c_op[512];
template <int NE>
__global__ void k_dfma_const(double* out) {
  double acc[NE], x[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) { acc[e] = 0; x[e] = threadIdx.x * 1e-3 + e; }
  for (int it = 0; it < ITERS / 32; ++it) {
#pragma unroll
    for (int j = 0; j < 64; ++j) {
#pragma unroll
      for (int e = 0; e < NE; ++e) { acc[e] = fma(c_op[2 * j], x[e], acc[e]); x[e] = fma(c_op[2 * j + 1], acc[e], x[e]); }
    }
  }
  double s = 0;
#pragma unroll
  for (int e = 0; e < NE; ++e) s += acc[e] + x[e];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma16816(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}
__device__ __forceinline__ void dmma1684(double (&c)[4], double a0, double a1, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b));
}

__global__ void k_dmma884(double* out, double a, double b) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = threadIdx.x; c[i][1] = i; }
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma884(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
__global__ void k_dmma1684(double* out, double a, double b) {
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = threadIdx.x + j + 7 * i;  // distinct chains (identical ones are merged by ptxas)
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) dmma1684(c[i], a, b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.678) out[0] = s;
}
__global__ void k_dmma16816(double* out, double a, double b) {
  double c[4][4], av[8], bv[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) av[i] = a + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) bv[i] = b + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = threadIdx.x + j + 7 * i;  // distinct chains (identical ones are merged by ptxas)
  for (int it = 0; it < ITERS / 16; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) dmma16816(c[i], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.678) out[0] = s;
}
// mixed: DMMA m8n8k4 and DFMA interleaved in one loop
__global__ void k_mixed(double* out, double a, double b) {
  double c[4][2], acc[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) { c[i][0] = threadIdx.x; c[i][1] = i; }
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) dmma884(c[i][0], c[i][1], a, b);
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}

template <class F>
float timeit(F f, int reps = 5) {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0)); f(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"device\":\"%s\",\"sms\":%d,\"clock_khz\":%d,\"l2_bytes\":%d}\n", p.name, sms, clk, p.l2CacheSize);
  double* out; CK(cudaMalloc(&out, 64));
  double* gop; CK(cudaMalloc(&gop, 4096 * 8)); CK(cudaMemset(gop, 0, 4096 * 8));
  double hop[512]; for (int i = 0; i < 512; ++i) hop[i] = 1e-3 * i; CK(cudaMemcpyToSymbol(c_op, hop, sizeof(hop)));
  for (int bs : {128, 256, 512}) {
    for (int bpsm : {4, 8, 16}) {
      int grid = sms * bpsm;
      if (bs * bpsm > 2048) continue;
      float ms = timeit([&] { k_dfma<<<grid, bs>>>(out, 1.0000001, 1e-9); });
      double fl = 2.0 * 8 * ITERS * (double)grid * bs;
      printf("{\"kern\":\"dfma_rr\",\"bs\":%d,\"grid\":%d,\"tflops\":%.3f}\n", bs, grid, fl / ms / 1e9);
    }
  }
  {
    int grid = sms * 4, bs = 256;
    float ms = timeit([&] { k_dfma_lds<1><<<grid, bs>>>(out, gop); });
    printf("{\"kern\":\"dfma_lds128_bcast_ne1\",\"tflops\":%.3f}\n", 2.0 * 2 * 1 * 16 * (ITERS / 8) * (double)grid * bs / ms / 1e9);
    ms = timeit([&] { k_dfma_lds<2><<<grid, bs>>>(out, gop); });
    printf("{\"kern\":\"dfma_lds128_bcast_ne2\",\"tflops\":%.3f}\n", 2.0 * 2 * 2 * 16 * (ITERS / 8) * (double)grid * bs / ms / 1e9);
    ms = timeit([&] { k_dfma_lds<4><<<grid, bs>>>(out, gop); });
    printf("{\"kern\":\"dfma_lds128_bcast_ne4\",\"tflops\":%.3f}\n", 2.0 * 2 * 4 * 16 * (ITERS / 8) * (double)grid * bs / ms / 1e9);
    ms = timeit([&] { k_dfma_const<1><<<grid, bs>>>(out); });
    printf("{\"kern\":\"dfma_const_ne1\",\"tflops\":%.3f}\n", 2.0 * 2 * 1 * 64 * (ITERS / 32) * (double)grid * bs / ms / 1e9);
    ms = timeit([&] { k_dfma_const<2><<<grid, bs>>>(out); });
    printf("{\"kern\":\"dfma_const_ne2\",\"tflops\":%.3f}\n", 2.0 * 2 * 2 * 64 * (ITERS / 32) * (double)grid * bs / ms / 1e9);
    ms = timeit([&] { k_dfma_const<4><<<grid, bs>>>(out); });
    printf("{\"kern\":\"dfma_const_ne4\",\"tflops\":%.3f}\n", 2.0 * 2 * 4 * 64 * (ITERS / 32) * (double)grid * bs / ms / 1e9);
  }
  for (int bpsm : {4, 8}) {
    int grid = sms * bpsm, bs = 256;
    float ms = timeit([&] { k_dmma884<<<grid, bs>>>(out, 1.0000001, 1e-9); });
    double warps = (double)grid * bs / 32;
    printf("{\"kern\":\"dmma_m8n8k4\",\"grid\":%d,\"tflops\":%.3f}\n", grid, 2.0 * 256 * 8 * (ITERS / 4) * warps / ms / 1e9);
    ms = timeit([&] { k_dmma1684<<<grid, bs>>>(out, 1.0000001, 1e-9); });
    printf("{\"kern\":\"dmma_m16n8k4\",\"grid\":%d,\"tflops\":%.3f}\n", grid, 2.0 * 512 * 4 * (ITERS / 4) * warps / ms / 1e9);
    ms = timeit([&] { k_dmma16816<<<grid, bs>>>(out, 1.0000001, 1e-9); });
    printf("{\"kern\":\"dmma_m16n8k16\",\"grid\":%d,\"tflops\":%.3f}\n", grid, 2.0 * 2048 * 4 * (ITERS / 16) * warps / ms / 1e9);
    ms = timeit([&] { k_mixed<<<grid, bs>>>(out, 1.0000001, 1e-9); });
    double fl = (2.0 * 256 * 4 * (ITERS / 4)) * warps + 2.0 * 32 * 8 * 4 * (ITERS / 4) * warps;
    printf("{\"kern\":\"mixed_dmma884_dfma\",\"grid\":%d,\"tflops\":%.3f}\n", grid, fl / ms / 1e9);
  }
  {
    size_t n = (size_t)1 << 27;  // 2^27 double2 = 2 GiB per buffer
    double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
    CK(cudaMemset(a, 0, n * 16));
    float ms = timeit([&] { k_copy<<<sms * 8, 512>>>(a, b, n); });
    printf("{\"kern\":\"copy_f64x2\",\"gbs_rw\":%.1f}\n", 2.0 * n * 16 / ms / 1e6);
    ms = timeit([&] { CK(cudaMemcpyAsync(b, a, n * 16, cudaMemcpyDeviceToDevice)); });
    printf("{\"kern\":\"cudaMemcpy_d2d\",\"gbs_rw\":%.1f}\n", 2.0 * n * 16 / ms / 1e6);
  }
  return 0;
}
