// Gather variant of the SIPDG operator for low degree (variant 5, N <= 3).  Paper: arXiv:1801.00246;
// same formulation as kernels.cuh.  At N <= 2 an element row is 24-48 bytes and the operator costs
// ~100-700 flop per element, so the path is bound by HBM; staging element blocks in shared memory
// (k_pipe, k_tpe) spends more on gathering small ghost rows than the arithmetic costs.  Here one
// thread owns one element and reads everything it needs straight from global memory (P:394's
// "one thread to one element" mapping): its own row and geometry records, and per interior face the
// neighbour's row and chain-rule record (L1/L2 hits: the neighbour is a nearby element in Morton order),
// from which it recomputes the neighbour's normal-derivative trace on the shared face only.
// The operators are compile-time indices into __constant__ memory (c_tpe, cops.cuh).
//   volume:  Au = Sr^T w_r + Ss^T w_s,  w = J G (Dr u, Ds u)          (Alg. AxG)
//   faces:   + (LIFT_f^T Sr)^T c_r delta + (LIFT_f^T Ss)^T c_s delta - E_f (sJ g)  (Alg. AxKernel)
//   PCG pass A: p_k = z + beta p_{k-1} formed for the own and the neighbour rows (one FMA, identical
//   everywhere), p_k and the deferred x update written for the own row, p.Ap reduced.
#pragma once
#include "sipdg_split.cuh"
#include "cops.cuh"

namespace ipdg {

// threads per CTA of k_gather: small CTAs so register-heavy instantiations still fill an SM in steps
// of 4 warps


// neighbour element `n` seen through its face FP: its values and traces sJ n.grad u (its own outward
// normal) at the face nodes, in its own face order
template <int N, int FP>
__device__ __forceinline__ void gather_face(const double (&un)[TrT<N>::NP], double Grr, double Grs, double Gss,
                                            double (&uf)[N + 1], double (&tf)[N + 1]) {
  using T = TrT<N>;
  constexpr int NP = T::NP, NFP = N + 1;
  const double* C = c_tpe<N>;
#pragma unroll
  for (int k = 0; k < NFP; ++k) {
    const int i = fmask_cf<N>(FP, k);
    double ur = 0.0, us = 0.0;
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      ur = fma(C[T::O_DR + i * NP + j], un[j], ur);
      us = fma(C[T::O_DS + i * NP + j], un[j], us);
    }
    const double wr = Grr * ur + Grs * us, ws = Grs * ur + Gss * us;
    tf[k] = (FP == 0) ? -ws : (FP == 1) ? wr + ws : -wr;
    uf[k] = un[i];
  }
}

template <int N, int MODE, bool LAM>
__global__ void __launch_bounds__(kGatherThreads) k_gather(AxArgs a) {
  using T = TrT<N>;
  constexpr int NP = T::NP, NFP = T::NFP;
  constexpr bool PCG = (MODE == MODE_PCG_A);
  __shared__ double red[32 * 3];
  const double* C = c_tpe<N>;
  const int64_t K = a.K;
  PcgDecision d;
  double* pnew = nullptr;
  const double* pold = nullptr;
  const double* U = a.u;
  if (PCG) {
    PcgState* st = a.st;
    if (st->stop_iter >= 0) return;
    d = pcg_decide(st);
    pnew = (d.k & 1) ? a.p_odd : a.p_even;
    pold = (d.k & 1) ? a.p_even : a.p_odd;
    U = a.z;
    if (d.stop) {
      const int64_t n = K * NP;
      for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (d.zero_x) a.x[i] = 0.0;
        else if (d.do_xupd) a.x[i] += d.alpha_prev * pold[i];
      }
      double v[1] = {0.0}, out[1];
      if (grid_reduce<1>(v, red, a.partials, a.counter, out)) {
        st->stop_iter = d.k - 1;
        st->status = d.new_status;
        st->final_rr = d.rrB;
        if (d.first) st->bb = d.bbv;
      }
      return;
    }
  }
  const bool with_p = PCG && !d.first;
  const double beta = d.beta;
  // operand row of element n (PCG: p_k = z + beta p_{k-1}, one FMA -- identical for the own row and as
  // a neighbour's; halo ghosts n >= K hold p_k already)
  auto load_row = [&](int64_t n, double (&v)[NP]) {
    if (n >= K) {
      const double* h = a.halo_p + (n - K) * NP;
#pragma unroll
      for (int i = 0; i < NP; ++i) v[i] = h[i];
    } else {
      const double* src = U + n * NP;
      const double* po = pold + n * NP;
#pragma unroll
      for (int i = 0; i < NP; ++i) v[i] = with_p ? fma(beta, po[i], src[i]) : src[i];
    }
  };
  // one element per thread, no grid-stride loop: a loop would let the compiler hoist the (loop-invariant)
  // operator constants into registers and spill them.  Measured alternatives that were slower on C3:
  // staging the block's rows through shared memory for coalesced access (N = 1: 45 -> 74 us) and raw
  // geometry with the factors recomputed per thread (45 -> 59 us).
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double dot = 0.0;
  if (e < K) {
    double u[NP];
    load_row(e, u);
    if (PCG) {  // own row: p_k and the deferred x update x += alpha_{k-1} p_{k-1}
#pragma unroll
      for (int i = 0; i < NP; ++i) {
        const int64_t g = e * NP + i;
        pnew[g] = u[i];
        if (d.do_xupd) a.x[g] = fma(d.alpha_prev, pold[g], a.x[g]);
      }
    }
    const double4 gg = a.gG[e];  // k_geofacs records
    const double Grr = gg.x, Grs = gg.y, Gss = gg.z, J = gg.w;
    double wr[NP], ws[NP];
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      double ur = 0.0, us = 0.0;
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        ur = fma(C[T::O_DR + i * NP + j], u[j], ur);
        us = fma(C[T::O_DS + i * NP + j], u[j], us);
      }
      wr[i] = Grr * ur + Grs * us;
      ws[i] = Grs * ur + Gss * us;
    }
    double out[NP];
#pragma unroll
    for (int n = 0; n < NP; ++n) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < NP; ++i) {
        s = fma(C[T::O_SR + i * NP + n], wr[i], s);
        s = fma(C[T::O_SS + i * NP + n], ws[i], s);
      }
      out[n] = s;
    }
    const int4 nb = a.nbg[e];
    const double* gf = a.gF + e * kGF;
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      const int fl = (nb.w >> (4 * f)) & 15;
      const int fp = fl & 3, bc = fl >> 2;
      const double cr = gf[3 * f], cs = gf[3 * f + 1], stau = gf[3 * f + 2];
      // own values and traces sJ n-.grad u- on face f
      double um[NFP], tm[NFP];
#pragma unroll
      for (int k = 0; k < NFP; ++k) {
        const int i = fmask_cf<N>(f, k);
        um[k] = u[i];
        tm[k] = (f == 0) ? -ws[i] : (f == 1) ? wr[i] + ws[i] : -wr[i];
      }
      double up[NFP], tp[NFP];  // exterior values / traces in own face order
      if (bc == 0) {  // interior: the neighbour's row, recomputed trace on its face fp (R3)
        const int64_t n = (f == 0) ? nb.x : (f == 1) ? nb.y : nb.z;
        double un[NP];
        load_row(n, un);
        const double4 gn = a.gG[n];
        double uf[NFP], tf[NFP];
        if (fp == 0) gather_face<N, 0>(un, gn.x, gn.y, gn.z, uf, tf);
        else if (fp == 1) gather_face<N, 1>(un, gn.x, gn.y, gn.z, uf, tf);
        else gather_face<N, 2>(un, gn.x, gn.y, gn.z, uf, tf);
        const bool flip = (f == 2) == (fp == 2);
#pragma unroll
        for (int k = 0; k < NFP; ++k) {
          up[k] = flip ? uf[NFP - 1 - k] : uf[k];
          tp[k] = flip ? tf[NFP - 1 - k] : tf[k];
        }
      } else {  // boundary: mirror the own trace (R7)
#pragma unroll
        for (int k = 0; k < NFP; ++k) {
          up[k] = um[k];
          tp[k] = tm[k];
        }
      }
      double dr[NFP], ds[NFP], fg[NFP];
#pragma unroll
      for (int k = 0; k < NFP; ++k) {
        const double delta = ((bc == 1) ? -up[k] : up[k]) - um[k];  // paper jump
        const double tq = (bc == 1) ? tp[k] : -tp[k];                // sJ n-.grad u+
        dr[k] = cr * delta;
        ds[k] = cs * delta;
        fg[k] = -0.5 * (tm[k] + tq) - stau * delta;                  // -sJ (n.{grad u} + tau delta)
      }
#pragma unroll
      for (int n = 0; n < NP; ++n) {
        double s = out[n];
#pragma unroll
        for (int k = 0; k < NFP; ++k) {
          const int fk = f * NFP + k;
          s = fma(C[T::O_LSR + fk * NP + n], dr[k], s);
          s = fma(C[T::O_LSS + fk * NP + n], ds[k], s);
        }
        out[n] = s;
      }
#pragma unroll
      for (int kk = 0; kk < NFP; ++kk) {  // face mass on the face rows
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < NFP; ++m) s = fma(C[T::O_M1D + kk * NFP + m], fg[m], s);
        out[fmask_cf<N>(f, kk)] += s;
      }
    }
    if (LAM) {
      const double lj = a.lambda * J;
#pragma unroll
      for (int n = 0; n < NP; ++n) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < NP; ++j) s = fma(C[T::O_M + n * NP + j], u[j], s);
        out[n] = fma(lj, s, out[n]);
      }
    }
#pragma unroll
    for (int n = 0; n < NP; ++n) {
      a.Au[e * NP + n] = out[n];
      if (PCG) dot += u[n] * out[n];
    }
  }
  if (PCG) {
    double v[1] = {dot}, outr[1];
    if (grid_reduce<1>(v, red, a.partials, a.counter, outr)) {
      a.st->red_A = outr[0];
      a.st->rho_hist[(d.k - 1) & 3] = d.rhoB;
      if (d.first) a.st->bb = d.bbv;
    }
  }
}

}  // namespace ipdg
