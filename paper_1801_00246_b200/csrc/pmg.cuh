// Matrix-free p-multigrid preconditioner kernels (R22-R26).
// The level operators are the library's own SIPDG Ax at each degree (child contexts); these kernels are
// the element-wise transfers, the Chebyshev smoother's vector steps and the reductions around them.
// Every kernel takes the PCG state `gate` (or null) and does nothing once the solve has stopped, so the
// cycles captured in an iteration graph after convergence cost only their (idle) launches.
#pragma once
#include "sipdg_kernels.cuh"

namespace ipdg {

__device__ __forceinline__ bool gated(const PcgState* g) { return g && g->stop_iter >= 0; }

// R26: the degree-1 level (no AMG tail) -- 16 Chebyshev steps over [1.1 lmax / 250, 1.1 lmax]
constexpr int kPmgCoarseSteps = 16;
constexpr double kPmgCoarseRatio = 250.0;

// uf (+)= P uc element by element: uf[e][i] = sum_j I[i][j] uc[e][j]   (R23, I row-major npf x npc)
static __global__ void k_prolong(int64_t K, int npf, int npc, const double* __restrict__ I, const double* __restrict__ uc,
                                 double* __restrict__ uf, int add, const PcgState* gate) {
  if (gated(gate)) return;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= K * npf) return;
  const int64_t e = t / npf;
  const int i = (int)(t - e * npf);
  const double* ur = uc + e * npc;
  const double* Ir = I + i * npc;
  double s = 0.0;
  for (int j = 0; j < npc; ++j) s = fma(Ir[j], ur[j], s);
  uf[t] = add ? uf[t] + s : s;
}

// rc = P^T rf element by element: rc[e][j] = sum_i I[i][j] rf[e][i]; with Af != null the fine residual
// rf - Af is formed on the fly (the pre-smoothed residual b - A x of the V-cycle, never stored)
static __global__ void k_restrict(int64_t K, int npf, int npc, const double* __restrict__ I, const double* __restrict__ rf,
                                  const double* __restrict__ Af, double* __restrict__ rc, const PcgState* gate) {
  if (gated(gate)) return;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= K * npc) return;
  const int64_t e = t / npc;
  const int j = (int)(t - e * npc);
  const double* rr = rf + e * npf;
  const double* ar = Af ? Af + e * npf : nullptr;
  double s = 0.0;
  for (int i = 0; i < npf; ++i) s = fma(I[i * npc + j], ar ? rr[i] - ar[i] : rr[i], s);
  rc[t] = s;
}

// Chebyshev step 0 from x = 0 (R24): d = D^{-1} b / theta, x = d.  With Ab != null the right-hand side is
// the residual b - Ab, formed here and stored in r (the post-smoother of the V-cycle)
static __global__ void k_cheb0(int64_t n, const double* __restrict__ b, const double* __restrict__ Ab,
                               double* __restrict__ r, const double* __restrict__ dinv, double inv_theta,
                               double* __restrict__ x, double* __restrict__ d, const PcgState* gate) {
  if (gated(gate)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double bi = b[i];
    if (Ab) {
      bi = bi - Ab[i];
      r[i] = bi;
    }
    const double v = dinv[i] * bi * inv_theta;
    d[i] = v;
    x[i] = v;
  }
}

// Chebyshev step 1 (R24): d = c1 d + c2 D^{-1} (b - A x), x += d   (Ax = A x, from the level's ipdg Ax).
// With acc != null (the post-smoother's last step) also acc += x, the V-cycle's correction of the level
// iterate; with rdot != null (level 0) the PCG's rho = rdot . acc is reduced into the state (red_B[0])
static __global__ void __launch_bounds__(256) k_cheb1(int64_t n, const double* __restrict__ b, const double* __restrict__ Ax,
                               const double* __restrict__ dinv, double c1, double c2, double* __restrict__ x,
                               double* __restrict__ d, double* __restrict__ acc, const double* __restrict__ rdot,
                               PcgState* st, double* partials, unsigned int* counter, const PcgState* gate) {
  __shared__ double red[32 * 3];
  if (gated(gate)) return;
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = fma(c1, d[i], c2 * dinv[i] * (b[i] - Ax[i]));
    d[i] = v;
    const double xi = x[i] + v;
    x[i] = xi;
    if (acc) {
      const double ai = acc[i] + xi;
      acc[i] = ai;
      if (rdot) s = fma(rdot[i], ai, s);
    }
  }
  if (rdot) {
    double vv[1] = {s}, o[1];
    if (grid_reduce<1>(vv, red, partials, counter, o)) st->red_B[0] = o[0];
  }
}

// deterministic dot product u.v -> out[0] (and, with st, rho = r.z of the PCG state: red_B[0])
static __global__ void __launch_bounds__(256) k_dot(int64_t n, const double* __restrict__ u, const double* __restrict__ v,
                                                    double* out, PcgState* st, double* partials, unsigned int* counter) {
  __shared__ double red[32 * 3];
  if (st && st->stop_iter >= 0) return;
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s = fma(u[i], v[i], s);
  double vv[1] = {s}, o[1];
  if (grid_reduce<1>(vv, red, partials, counter, o)) {
    if (out) out[0] = o[0];
    if (st) st->red_B[0] = o[0];
  }
}

// R24 power iteration: the fixed start vector v_i = ((7919 i) mod 1009) / 1009 - 1/2
static __global__ void k_pmg_start(int64_t n, double* __restrict__ v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (double)((7919 * i) % 1009) / 1009.0 - 0.5;
}

// w = D^{-1} (A v)
static __global__ void k_scale(int64_t n, const double* __restrict__ dinv, const double* __restrict__ Av, double* __restrict__ w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    w[i] = dinv[i] * Av[i];
}

// v = w / nw (nw read from device memory)
static __global__ void k_normalize(int64_t n, const double* __restrict__ w, const double* nw, double* __restrict__ v) {
  const double s = 1.0 / sqrt(nw[0]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = w[i] * s;
}

}  // namespace ipdg
