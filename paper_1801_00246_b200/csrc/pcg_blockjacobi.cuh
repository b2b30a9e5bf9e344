// Block-Jacobi preconditioner of the screened Poisson solve: "the scaled inverse
// mass matrix on each element" for A = -L + lambda (Eq. ellipticOp1), z_e = (lambda J^e M)^{-1} r_e
// = M^{-1} r_e / (lambda J^e) (M^e = J^e M, Eq. elementOps).
//   INIT:   r = b - A x0, z = P r, partial (r.z, r.r, b.b)            (replaces k_pcg_init)
//   update: r -= alpha A p, z = P r, partial (r.z, r.r); breakdown test  (replaces k_pcg_b; with x != null
//           also x += alpha p_k, as k_pcg_b)
// One thread per DOF of a chunk of E = 256 / Np elements: the updated residual rows and M^{-1}
// (staged once per CTA, odd row stride Np + 1 - Np % 2 against bank conflicts) are read from shared
// memory, z_i = sum_j Minv[i][j] r_j; few registers, so several CTAs share an SM.
#pragma once
#include "sipdg_kernels.cuh"

namespace ipdg {

template <int N, bool INIT>
__global__ void __launch_bounds__(256, 3) k_pcg_bj(int64_t K, const double* in0, const double* __restrict__ in1,
                                                double* r, double* __restrict__ z,
                                                const double4* __restrict__ gG, const double* __restrict__ Minv,
                                                double lambda, PcgState* st, double* partials, unsigned int* counter,
                                                double* __restrict__ x, const double* p_even, const double* p_odd) {
  constexpr int NP = Tr<N>::NP, EPB = 256 / NP, ACT = EPB * NP, MS = NP | 1;
  __shared__ double rs[ACT];
  __shared__ double ms[NP * MS];
  __shared__ double red[32 * 3];
  const int t = threadIdx.x;
  const int el = t / NP, i = t - el * NP;
  const bool active = t < ACT;
  double alpha = 0.0;
  const double* p = nullptr;
  if (!INIT) {
    if (st->stop_iter >= 0) return;
    const long long k = st->it + 1;
    p = (k & 1) ? p_odd : p_even;
    const double sigma = st->red_A;
    const double rho = st->rho_hist[(k - 1) & 3];
    if (!(sigma > 0.0)) {  // breakdown: p^T A p <= 0 (or NaN)
      double v[2] = {0.0, 0.0}, out[2];
      if (grid_reduce<2>(v, red, partials, counter, out)) {
        st->stop_iter = k;
        st->status = -4;
        st->final_rr = st->red_B[1];
        st->it = k;
      }
      return;
    }
    alpha = rho / sigma;
  }
  for (int q = t; q < NP * NP; q += 256) ms[(q / NP) * MS + q % NP] = Minv[q];
  const double* mrow = ms + i * MS;
  double rz = 0.0, rr = 0.0, bb = 0.0;
  for (int64_t e0 = (int64_t)blockIdx.x * EPB; e0 < K; e0 += (int64_t)gridDim.x * EPB) {
    const int64_t e = e0 + el;
    const bool ok = active && e < K;
    const int64_t g = e * NP + i;
    double rv = 0.0;
    if (ok) {
      if (INIT) {
        const double bi = in0[g];
        rv = bi - in1[g];
        bb += bi * bi;
      } else {
        if (x) x[g] = fma(alpha, p[g], x[g]);  // x += alpha_k p_k when pass A does not (defer_x = 0)
        rv = in0[g] - alpha * in1[g];
      }
      r[g] = rv;
    }
    __syncthreads();  // the previous chunk's rows are consumed
    if (active) rs[t] = rv;
    __syncthreads();
    if (ok) {
      const double* row = rs + el * NP;
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < NP; ++j) s = fma(mrow[j], row[j], s);
      const double zi = s / (lambda * gG[e].w);
      z[g] = zi;
      rz += rv * zi;
      rr += rv * rv;
    }
  }
  if (INIT) {
    double v[3] = {rz, rr, bb}, out[3];
    if (grid_reduce<3>(v, red, partials, counter, out)) {
      st->red_B[0] = out[0];
      st->red_B[1] = out[1];
      st->red_B[2] = out[2];
    }
  } else {
    double v[2] = {rz, rr}, out[2];
    if (grid_reduce<2>(v, red, partials, counter, out)) {
      st->red_B[0] = out[0];
      st->red_B[1] = out[1];
      st->it = st->it + 1;
    }
  }
}

}  // namespace ipdg
