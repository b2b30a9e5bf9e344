// Split two-kernel variant of the SIPDG operator for high degree (N >= 6 by default).
// Paper: arXiv:1801.00246.  Same formulation as kernels.cuh / sipdg_kernels.cuh.
//
// The fused kernel keeps the DMMA operator tables (37 + 69 KB at N = 8) and a block of element
// data in shared memory at once, which leaves one CTA of 4 warps per SM at N >= 7.  Like the
// paper's two-kernel design (local gradient kernel, Alg. AxG, then the SIPDG kernel,
// Alg. AxKernel) the work is split so each kernel holds one table:
//   k_grad:  W = [w_r | w_s] = J G [D_r u | D_s u] for own and halo-ghost elements -> global
//            (the scaled normal derivatives on the faces are -w_s, w_r + w_s, -w_r)
//   k_flux:  per own face node: jump, mirrored traces, flux from W and u of both sides (global,
//            the neighbour rows come from L2), then Au = [w_r | w_s | face block] x [Sr; Ss;
//            LIFT^T Sr; LIFT^T Ss; E^T] (+ lambda J u M) on DMMA, and p.Ap in PCG pass A.
// Every warp works on its own 8-element tile; there is no block-wide synchronisation after the
// table staging.  Extra traffic: W written and read once (32 Np B/element).
#pragma once
#include "kernels.cuh"

namespace ipdg {

struct SplitArgs {
  int64_t K, H;
  const double4* gG;     // [K + H] (J G_rr, J G_rs, J G_ss, J) (k_geofacs)
  const double* gF;      // [K][kGF] per face (1/2 sJ n.grad r, 1/2 sJ n.grad s, sJ tau)
  int64_t ebeg, eend;    // k_grad: element rows [ebeg, eend) of the K + H (own | halo) rows
  int stop_work;         // k_grad PCG: this launch applies the deferred x update when the loop stops
  const double4* geo;    // [K+H]
  const int4* nbg;       // [K] neighbour element per face (>= K: halo ghost) + flags (f' | bc << 2) << 4f in .w
  const double* tables;  // G | M | L | aux | M2 (natural w rows)
  double tau_c, lambda;
  const double* u;       // AX: operand rows [K]
  const double* halo;    // [H] ghost rows (AX: u, PCG: p_k)
  double* W2;            // [(K+H) x 2 Np]
  double* Au;
  const double* z;       // D^-1 r (or r)
  double* p_even;
  double* p_odd;
  double* x;
  PcgState* st;
  double* partials;
  unsigned int* counter;
};

template <int N>
struct TrS {
  using T = Tr<N>;
  static constexpr int W = 8;                             // warps per CTA (independent tiles)
  static constexpr int KCW2 = 2 * T::KCG;                  // natural w rows: w_r | w_s, NPK each
  static constexpr int TAB_M2 = (KCW2 + T::KCF) * T::NT * 32;
  static constexpr int AUX = T::NFP * T::NFP + (T::NF3 + 2 * T::NPN + 1) / 2;  // M1D + index ints (see build_tables)
  static constexpr int OFF_M2 = T::TAB_G + T::TAB_M + T::TAB_L + ((AUX + 1) & ~1);
};

// decisions of PCG pass A from the previous iteration's reductions (identical in every CTA)
struct PcgDecision {
  bool stop = false, first = false, zero_x = false, do_xupd = false;
  long long k = 0;
  int new_status = 0;
  double beta = 0.0, alpha_prev = 0.0, rhoB = 0.0, rrB = 0.0, bbv = 0.0;
};

__device__ __forceinline__ PcgDecision pcg_decide(const PcgState* st) {
  PcgDecision d;
  d.k = st->it + 1;
  d.first = (d.k == 1);
  d.rhoB = st->red_B[0];
  d.rrB = st->red_B[1];
  d.bbv = d.first ? st->red_B[2] : st->bb;
  if (d.first) {
    if (d.bbv == 0.0) { d.stop = true; d.zero_x = true; }
    else if (d.rrB <= st->tol2 * d.bbv) d.stop = true;
    else if (st->maxit == 0) { d.stop = true; d.new_status = 1; }
  } else {
    if (d.rrB <= st->tol2 * d.bbv) d.stop = true;
    else if (d.k - 1 >= st->maxit) { d.stop = true; d.new_status = 1; }
    d.alpha_prev = st->rho_hist[(d.k - 2) & 3] / st->red_A;
    d.do_xupd = true;
    d.beta = d.rhoB / st->rho_hist[(d.k - 2) & 3];
  }
  return d;
}

// ---------------------------------------------------------------- k_grad
template <int N, int MODE>
__global__ void __launch_bounds__(TrS<N>::W * 32) k_grad(SplitArgs a) {
  using T = Tr<N>;
  constexpr int NP = T::NP, NT = T::NT, SU = T::SU, KCG = T::KCG, W = TrS<N>::W;
  extern __shared__ __align__(16) double sm[];
  double* tabG = sm;
  double* stage = sm + T::TAB_G;  // per warp 8 x SU
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t K = a.K, KH = a.K + a.H;
  PcgDecision d;
  double* pnew = nullptr;
  const double* pold = nullptr;
  if (MODE == MODE_PCG_A) {
    if (a.st->stop_iter >= 0) return;
    d = pcg_decide(a.st);
    pnew = (d.k & 1) ? a.p_odd : a.p_even;
    pold = (d.k & 1) ? a.p_even : a.p_odd;
    if (d.stop) {  // deferred x update only; k_flux records the decision
      if (!a.stop_work) return;
      const int64_t n = K * NP;
      for (int64_t i = blockIdx.x * (int64_t)blockDim.x + tid; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (d.zero_x) a.x[i] = 0.0;
        else if (d.do_xupd) a.x[i] += d.alpha_prev * pold[i];
      }
      return;
    }
  }
  for (int i = 2 * tid; i < T::TAB_G; i += 2 * blockDim.x) cp_async16(sm + i, a.tables + i);
  cp_async_wait_all();
  double* st8 = stage + warp * 8 * SU;
  for (int i = lane; i < 8 * SU; i += 32) st8[i] = 0.0;
  __syncthreads();
  // rows [ebeg, eend): all K + H rows, or the own rows and then the halo rows (the latter after the
  // halo exchange, which the own rows overlap).  Software pipeline: the operand rows (PCG: z, p_{k-1}, x)
  // and the geometry record of tile t + stride are loaded into registers while tile t computes.
  constexpr int NPF = (8 * NP + 31) / 32;  // row values per lane for one 8-element tile
  // prefetching costs registers (occupancy): measured faster for PCG pass A at N = 6, 8 and for Ax at N = 8,
  // slower for Ax at N = 6 (C3: 636 -> 661 us), so Ax at N <= 6 loads each tile when it starts it
  constexpr bool PF = (MODE == MODE_PCG_A) || N >= 7;
  const int64_t ntiles = (a.eend - a.ebeg + 7) / 8;
  const int64_t tstride = (int64_t)gridDim.x * W;
  double pv[NPF], pp[NPF], px[NPF];
  double4 pg = make_double4(0, 0, 0, 0);
  auto fetch = [&](int64_t t) {
    const int64_t e0 = a.ebeg + 8 * t;
    const int nrow = (int)min((int64_t)8, a.eend - e0);
#pragma unroll
    for (int r = 0; r < NPF; ++r) {
      const int q = lane + 32 * r;
      pv[r] = pp[r] = px[r] = 0.0;
      if (q < nrow * NP) {
        const int el = q / NP, i = q - el * NP;
        const int64_t e = e0 + el;
        if (e >= K) {
          pv[r] = a.halo[(e - K) * NP + i];
        } else if (MODE == MODE_AX) {
          pv[r] = __ldg(a.u + e * NP + i);
        } else {
          const int64_t g = e * NP + i;
          pv[r] = __ldg(a.z + g);
          if (!d.first) pp[r] = pold[g];
          if (d.do_xupd) px[r] = a.x[g];
        }
      }
    }
    const int64_t e = e0 + (lane >> 2);
    if (e < a.eend) pg = a.gG[e];
  };
  int64_t t = (int64_t)blockIdx.x * W + warp;
  if (PF && t < ntiles) fetch(t);
  for (; t < ntiles; t += tstride) {
    const int64_t e0 = a.ebeg + 8 * t;
    const int nrow = (int)min((int64_t)8, a.eend - e0);
    if (!PF) fetch(t);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < NPF; ++r) {  // operand rows of the tile (contiguous for own rows)
      const int q = lane + 32 * r;
      if (q < nrow * NP) {
        const int el = q / NP, i = q - el * NP;
        const int64_t e = e0 + el;
        double v = pv[r];
        if (MODE == MODE_PCG_A && e < K) {
          const int64_t g = e * NP + i;
          v = pv[r] + d.beta * pp[r];
          pnew[g] = v;
          if (d.do_xupd) a.x[g] = px[r] + d.alpha_prev * pp[r];
        }
        st8[el * SU + i] = v;
      }
    }
    const double4 gr = pg;  // J G^T G from the setup records (k_geofacs)
    if (PF && t + tstride < ntiles) fetch(t + tstride);
    __syncwarp();
    double acc[2 * NT][2];
#pragma unroll
    for (int q = 0; q < 2 * NT; ++q) acc[q][0] = acc[q][1] = 0.0;
    const double* urow = st8 + (lane >> 2) * SU + (lane & 3);
#pragma unroll
    for (int kc = 0; kc < KCG; ++kc) {
      const double av = urow[4 * kc];
      const double* bt = tabG + kc * 2 * NT * 32 + lane;
#pragma unroll
      for (int q = 0; q < 2 * NT; ++q) dmma(acc[q][0], acc[q][1], av, bt[q * 32]);
    }
    const int64_t e = e0 + (lane >> 2);
    if (e < a.eend) {
      const double Grr = gr.x, Grs = gr.y, Gss = gr.z;
      double* wrow = a.W2 + e * 2 * NP;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = 8 * nt + 2 * (lane & 3) + h;
          if (i < NP) {
            const double ur = acc[nt][h], us = acc[NT + nt][h];
            wrow[i] = Grr * ur + Grs * us;
            wrow[NP + i] = Grs * ur + Gss * us;
          }
        }
    }
  }
}

// ---------------------------------------------------------------- k_flux
template <int N, int MODE, bool LAM>
__global__ void __launch_bounds__(TrS<N>::W * 32) k_flux(SplitArgs a) {
  using T = Tr<N>;
  using S = TrS<N>;
  constexpr int NP = T::NP, NFP = T::NFP, NF3 = T::NF3, NT = T::NT, KCG = T::KCG, KCF = T::KCF, KCM = T::KCM;
  constexpr int W = S::W, NQ = T::NQ;
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[32 * 3];
  double* tabM = sm;
  double* tabL = sm + S::TAB_M2;
  __shared__ int nidx[6 * NFP];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t K = a.K;
  PcgDecision d;
  const double* U = a.u;
  if (MODE == MODE_PCG_A) {
    if (a.st->stop_iter >= 0) return;
    d = pcg_decide(a.st);
    U = (d.k & 1) ? a.p_odd : a.p_even;  // p_k written by k_grad
    if (d.stop) {
      double v[1] = {0.0}, out[1];
      if (grid_reduce<1>(v, red, a.partials, a.counter, out)) {
        a.st->stop_iter = d.k - 1;
        a.st->status = d.new_status;
        a.st->final_rr = d.rrB;
        if (d.first) a.st->bb = d.bbv;
      }
      return;
    }
  }
  {
    const double* src = a.tables + S::OFF_M2;
    for (int i = 2 * tid; i < S::TAB_M2; i += 2 * blockDim.x) cp_async16(sm + i, src + i);
    if (LAM) {
      const double* srcl = a.tables + T::TAB_G + T::TAB_M;
      for (int i = 2 * tid; i < T::TAB_L; i += 2 * blockDim.x) cp_async16(tabL + i, srcl + i);
    }
    for (int q = tid; q < 6 * NFP; q += blockDim.x) {
      const int fp = q / (2 * NFP), fl = (q / NFP) & 1, kk = q % NFP;
      nidx[q] = fmask_cf<N>(fp, fl ? NFP - 1 - kk : kk);
    }
    cp_async_wait_all();
    __syncthreads();
  }
  int itab[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int fk = 4 * q + (lane & 3);
    const int f = fk / NFP, kk = fk - f * NFP;
    itab[q] = (fk < NF3) ? ((f << 24) | (kk << 16) | fmask_cf<N>(f, kk)) : -1;
  }
  double dot = 0.0;
  const int64_t ntiles = (K + 7) / 8;
  for (int64_t t = (int64_t)blockIdx.x * W + warp; t < ntiles; t += (int64_t)gridDim.x * W) {
    const int64_t e0 = 8 * t;
    const int64_t eraw = e0 + (lane >> 2);
    const bool valid = eraw < K;
    const int64_t e = valid ? eraw : e0;
    const int4 nb = a.nbg[e];
    // per-face coefficients (1/2 sJ n.grad r, 1/2 sJ n.grad s, sJ tau) from the setup records (k_geofacs):
    // lane (element, f < 3) loads face f, the others read it by shuffle
    double ccr = 0.0, ccs = 0.0, cst = 0.0;
    {
      const int f = lane & 3;
      if (f < 3) {
        const double* r = a.gF + e * kGF + 3 * f;
        ccr = r[0];
        ccs = r[1];
        cst = r[2];
      }
    }
    const double* uo = U + e * NP;
    const double* wo = a.W2 + e * 2 * NP;
    double far[NQ], fas[NQ], fag[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int it = itab[q];
      const int f = it >= 0 ? (it >> 24) : 0;
      const int src = (lane & ~3) | f;
      const double cr = __shfl_sync(0xffffffffu, ccr, src);
      const double cs = __shfl_sync(0xffffffffu, ccs, src);
      const double ct = __shfl_sync(0xffffffffu, cst, src);
      far[q] = fas[q] = fag[q] = 0.0;
      if (it >= 0) {
        const int kk = (it >> 16) & 255, i = it & 65535;
        const int fl = (nb.w >> (4 * f)) & 15;
        const int fp = fl & 3, bc = fl >> 2;
        const bool inner = (bc == 0);
        const int64_t n = (f == 0) ? nb.x : (f == 1) ? nb.y : nb.z;
        const int64_t pe = inner ? n : e;
        const int pf = inner ? fp : f;
        const int ip = inner ? nidx[(2 * fp + ((f == 2) == (fp == 2))) * NFP + kk] : i;
        const double upr = (pe >= K) ? a.halo[(pe - K) * NP + ip] : U[pe * NP + ip];
        const double* wn = a.W2 + pe * 2 * NP;
        const double um = uo[i];
        const double wro = wo[i], wso = wo[NP + i], wrn = wn[ip], wsn = wn[NP + ip];
        const double tm = (f == 0) ? -wso : (f == 1) ? wro + wso : -wro;
        const double tp = (pf == 0) ? -wsn : (pf == 1) ? wrn + wsn : -wrn;
        const double tq = (bc == 1) ? tp : -tp;
        const double delta = ((bc == 1) ? -upr : upr) - um;
        far[q] = cr * delta;
        fas[q] = cs * delta;
        fag[q] = -0.5 * (tm + tq) - ct * delta;
      }
    }
    double C[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) C[nt][0] = C[nt][1] = 0.0;
#pragma unroll
    for (int kc = 0; kc < KCG; ++kc) {  // w_r, w_s in natural node order
      const int k = 4 * kc + (lane & 3);
      const double ar = (k < NP) ? wo[k] : 0.0;
      const double as = (k < NP) ? wo[NP + k] : 0.0;
      const double* b0 = tabM + kc * NT * 32 + lane;
      const double* b1 = tabM + (KCG + kc) * NT * 32 + lane;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        dmma(C[j][0], C[j][1], ar, b0[j * 32]);
        dmma(C[j][0], C[j][1], as, b1[j * 32]);
      }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const double* b0 = tabM + (S::KCW2 + q) * NT * 32 + lane;
      const double* b1 = tabM + (S::KCW2 + NQ + q) * NT * 32 + lane;
      const double* b2 = tabM + (S::KCW2 + 2 * NQ + q) * NT * 32 + lane;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        dmma(C[j][0], C[j][1], far[q], b0[j * 32]);
        dmma(C[j][0], C[j][1], fas[q], b1[j * 32]);
        dmma(C[j][0], C[j][1], fag[q], b2[j * 32]);
      }
    }
    if (LAM) {
      const double lj = a.lambda * a.gG[e].w;  // lambda J
#pragma unroll
      for (int kc = 0; kc < KCM; ++kc) {
        const int k = 4 * kc + (lane & 3);
        const double av = (k < NP) ? lj * uo[k] : 0.0;
        const double* bt = tabL + kc * NT * 32 + lane;
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(C[j][0], C[j][1], av, bt[j * 32]);
      }
    }
    if (valid) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = 8 * nt + 2 * (lane & 3) + h;
          if (i < NP) {
            a.Au[e * NP + i] = C[nt][h];
            if (MODE == MODE_PCG_A) dot += uo[i] * C[nt][h];
          }
        }
    }
  }
  if (MODE == MODE_PCG_A) {
    double v[1] = {dot}, out[1];
    if (grid_reduce<1>(v, red, a.partials, a.counter, out)) {
      a.st->red_A = out[0];
      a.st->rho_hist[(d.k - 1) & 3] = d.rhoB;
      if (d.first) a.st->bb = d.bbv;
    }
  }
}

}  // namespace ipdg
