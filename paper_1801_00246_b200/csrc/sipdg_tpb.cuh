// Thread-per-element, block-staged SIPDG operator (variant 6, k_tpb).  Paper: arXiv:1801.00246;
// operator as kernels.cuh (Eqs. ellipticOp1/ellipticOp3; Alg. AxG, Alg. AxKernel
// P:542-603).  P:394's "one thread to one element" mapping, built for B200's FP64 datapath:
//
// * No tensor-core padding: every product is a DFMA whose operator entry is a compile-time index into
//   __constant__ memory (uniform-register operand), so the FP64 pipe does only useful work.
// * Face derivatives split into a tangential and a transverse part.  The restriction of u to a face
//   is the degree-N polynomial through its N+1 face nodes, so the derivative ALONG face f needs only
//   those values (D1D, N_fp^2); only the transverse derivative needs the whole row (T_f, N_fp x N_p).
//   face 0 (s = -1): d/dxi = d/dr, transverse d/ds;  face 1 (r + s = 0, xi = s): d/dxi = d/ds - d/dr,
//   transverse d/dr;  face 2 (r = -1): d/dxi = d/ds, transverse d/dr.  The lifted jump of Eq.
//   ellipticOp3, (LIFT_f^T S_r)^T c_r delta + (LIFT_f^T S_s)^T c_s delta = (c_r D_r,f + c_s D_s,f)^T M1D delta,
//   becomes a_f P_f delta + b_f scatter_f(Q delta), P_f = T_f^T M1D (N_p x N_fp), Q = D1D^T M1D.
//   Per element: 4N_p^2 (gradient form, N <= 5) or 3N_p^2 + 3(N_fp N_p + N_fp^2) (stiffness form
//   K_rr, K_rs + K_sr, K_ss, N >= 6) for the volume and own traces, plus 3(N_fp N_p + 2 N_fp^2) for the
//   lift and the face mass -- below F_min of the DMMA formulation.
// * Element blocks of E consecutive elements per CTA (one thread each).  Every own element writes its
//   face values and traces sJ n.grad u (outward) to shared memory; a neighbour inside the block reads
//   them there.  Neighbours outside the block are "ghost faces": a compact list per block (sorted by
//   the ghost's face index, so warps stay convergent) whose traces are recomputed on that face only
//   (N_fp N_p + N_fp^2 MACs each) by the first threads of the CTA.
// * Own rows arrive by one TMA bulk copy per block (cp.async.bulk + mbarrier); PCG pass A forms
//   p_k = z + beta p_{k-1} and the deferred x update in one coalesced pass; Au is written in place
//   over the staged rows and leaves by one bulk copy (cp.async.bulk shared -> global).
#pragma once
#include "sipdg_split.cuh"

namespace ipdg {

template <int N_>
struct TrB {
  static constexpr int N = N_;
  static constexpr int NP = (N + 1) * (N + 2) / 2, NFP = N + 1, NF3 = 3 * NFP;
#ifndef IPDG_TPB_R
#define IPDG_TPB_R 1
#endif
  // elements per thread: every operator entry loaded from the constant bank feeds R independent FMAs
  // (the constant path delivers ~8 B/clk/SM: one DFMA per entry caps the FP64 pipe near 50 %,
  // tools/micro_const.cu)
  static constexpr int R = IPDG_TPB_R;
  static constexpr int E = tpb_e(N);           // elements per CTA
  static constexpr int NTHR = E / R;
#ifndef IPDG_TPB_REGS
#define IPDG_TPB_REGS 0
#endif
  static constexpr int RCAP = IPDG_TPB_REGS > 0 ? IPDG_TPB_REGS : (R == 1 ? 128 : 255);  // register cap per thread
  static constexpr int MINB = 65536 / (RCAP * NTHR) > 0 ? 65536 / (RCAP * NTHR) : 1;
  static constexpr int TS = NF3 | 1;           // face-record stride per slot (odd: 16-byte accesses spread over banks)
  static constexpr bool FULLF = N <= 5;        // face loops fully unrolled (else the lift loop is rolled)
  // __constant__ layout (doubles), read in address order by the loops below.  64 KB bank per degree:
  // at N = 8 the lift goes through T_f^T (M1D delta) and there is no mass table (no lambda term).
  static constexpr bool BIG = N >= 8;
#ifndef IPDG_TPB_GRAD_MAX
#define IPDG_TPB_GRAD_MAX 5
#endif
  // volume: gradient form (Dr, Ds then Sr^T, Ss^T: 4 NP^2, own traces from the gradient) or stiffness
  // form (Krr, Krs, Kss: 3 NP^2 plus the own traces through the face-derivative split, fewer registers)
  static constexpr bool GRAD = N <= IPDG_TPB_GRAD_MAX;
  static constexpr int O_KRR = 0;                                  // [j][n] K_rr = Dr^T M Dr     | grad: [j][i] Dr[i][j]
  static constexpr int O_KRS = O_KRR + NP * NP;                    // [j][n] Dr^T M Ds + Ds^T M Dr | grad: [j][i] Ds[i][j]
  static constexpr int O_KSS = O_KRS + NP * NP;                    // [j][n] K_ss = Ds^T M Ds     | grad: [i][n] Sr[i][n]
  static constexpr int O_SS = O_KSS + NP * NP;                     //                             | grad: [i][n] Ss[i][n]
  static constexpr int O_DRT = O_KRR, O_DST = O_KRS, O_SR = O_KSS;
  static constexpr int O_TN = O_SS + (GRAD ? NP * NP : 0);         // [f][k][n] transverse derivative rows T_f[k][n]
  static constexpr int O_PT = O_TN + 3 * NFP * NP;                 // [f][k][n] (T_f^T M1D)[n][k]   (not BIG)
  static constexpr int O_QT = O_PT + (BIG ? 0 : 3 * NP * NFP);     // [k][m] (D1D^T M1D)[m][k]      (not BIG)
  static constexpr int O_M1D = O_QT + (BIG ? 0 : NFP * NFP);       // [m][k] (symmetric)
  static constexpr int O_D1DT = O_M1D + NFP * NFP;                 // [m][k] = D1D[k][m], d/dxi on the face nodes
  static constexpr int O_M = O_D1DT + NFP * NFP;                   // [j][n] reference mass (lambda term, not BIG)
  static constexpr int TOTAL = O_M + (BIG ? 0 : NP * NP);
  static constexpr bool HAS_LAM = !BIG;
#ifndef IPDG_TPB_UNR
#define IPDG_TPB_UNR 0
#endif
  static constexpr int UNR = IPDG_TPB_UNR > 0 ? IPDG_TPB_UNR : NP;  // unroll of the row loops (NP: full)
};

template <int N>
__constant__ double c_tpb[TrB<N>::TOTAL];

// shared-memory layout in doubles: rows [E x NP] (+1 pad) | face records ft [E x TS] double2 |
// ghost-face records gft [gmax x NFP] double2 | mbarrier
template <int N>
struct TpbLayout {
  using T = TrB<N>;
  static constexpr int ROWS = 0;
  static constexpr int FT = ((T::E * T::NP + 1) + 1) & ~1;
  // The face-record region first holds the staged p_{k-1} and x rows (PCG pass A), consumed by the
  // formation pass before the face records are written (a block barrier in between).
  static constexpr int FTN = (2 * T::E * T::TS > 2 * T::E * T::NP ? 2 * T::E * T::TS : 2 * T::E * T::NP);
  __host__ __device__ static int gft(int, bool) { return FT + FTN; }
  __host__ __device__ static int mbar(int gmax, bool pcg) { return gft(gmax, pcg) + 2 * gmax * T::NFP; }
  __host__ __device__ static int total(int gmax, bool pcg) { return mbar(gmax, pcg) + 2; }
};

__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// trace sJ n.grad u (outward normal) at the N_fp nodes of face FP of an element with row u and chain-rule
// record (J G_rr, J G_rs, J G_ss): tangential derivative from the face values, transverse from the row
template <int N, int FP, int RR, class Row>
__device__ __forceinline__ void face_trace(const Row& u, const double* Grr, const double* Grs, const double* Gss,
                                           double (&tf)[RR][N + 1]) {
  using T = TrB<N>;
  constexpr int NP = T::NP, NFP = T::NFP;
  const double* C = c_tpb<N>;
  double ut[RR][NFP], ux[RR][NFP];
#pragma unroll
  for (int r = 0; r < RR; ++r)
#pragma unroll
    for (int k = 0; k < NFP; ++k) ut[r][k] = ux[r][k] = 0.0;
#pragma unroll(T::UNR)
  for (int j = 0; j < NP; ++j) {  // transverse derivative: the whole row
    double uj[RR];
#pragma unroll
    for (int r = 0; r < RR; ++r) uj[r] = u(r, j);
#pragma unroll
    for (int k = 0; k < NFP; ++k)
#pragma unroll
      for (int r = 0; r < RR; ++r) ut[r][k] = fma(C[T::O_TN + (FP * NFP + k) * NP + j], uj[r], ut[r][k]);
  }
#pragma unroll
  for (int m = 0; m < NFP; ++m) {  // tangential derivative: the face values
    double um[RR];
#pragma unroll
    for (int r = 0; r < RR; ++r) um[r] = u(r, fmask_cf<N>(FP, m));
#pragma unroll
    for (int k = 0; k < NFP; ++k)
#pragma unroll
      for (int r = 0; r < RR; ++r) ux[r][k] = fma(C[T::O_D1DT + m * NFP + k], um[r], ux[r][k]);
  }
#pragma unroll
  for (int r = 0; r < RR; ++r)
#pragma unroll
    for (int k = 0; k < NFP; ++k) {
      if (FP == 0) tf[r][k] = -(Grs[r] * ux[r][k] + Gss[r] * ut[r][k]);                                // -w_s
      else if (FP == 1) tf[r][k] = (Grr[r] + Grs[r]) * ut[r][k] + (Grs[r] + Gss[r]) * (ux[r][k] + ut[r][k]);  // w_r + w_s
      else tf[r][k] = -(Grr[r] * ut[r][k] + Grs[r] * ux[r][k]);                                       // -w_r
    }
}

// value and trace of a ghost element on its face FP, in that face's node order
template <int N, int FP>
__device__ __forceinline__ void ghost_face(const double (&un)[TrB<N>::NP], double4 gn, double2* go) {
  constexpr int NFP = N + 1;
  double tf[1][NFP];
  auto ur = [&](int, int j) { return un[j]; };
  face_trace<N, FP, 1>(ur, &gn.x, &gn.y, &gn.z, tf);
#pragma unroll
  for (int k = 0; k < NFP; ++k) go[k] = make_double2(un[fmask_cf<N>(FP, k)], tf[0][k]);
}

template <int N, int MODE, bool LAM>
__global__ void __launch_bounds__(TrB<N>::NTHR, TrB<N>::MINB) k_tpb(AxArgs a, int gmax) {
  using T = TrB<N>;
  using L = TpbLayout<N>;
  constexpr int NP = T::NP, NFP = T::NFP, E = T::E, TS = T::TS, NTHR = T::NTHR, R = T::R;
  constexpr bool PCG = (MODE == MODE_PCG_A);
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[32 * 3];
  double* rows = sm + L::ROWS;
  double2* ft = reinterpret_cast<double2*>(sm + L::FT);
  double2* gft = reinterpret_cast<double2*>(sm + L::gft(gmax, PCG));
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(sm + L::mbar(gmax, PCG));
  const double* C = c_tpb<N>;
  const int tid = threadIdx.x;
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
    if (d.stop) {  // the deferred x update of ALL rows (grid-stride): a split pass A stops in its first launch
      const int64_t n = K * NP;
      for (int64_t i = blockIdx.x * (int64_t)NTHR + tid; i < n; i += (int64_t)gridDim.x * NTHR) {
        if (d.zero_x) a.x[i] = 0.0;
        else if (d.do_xupd && a.defer_x) a.x[i] += d.alpha_prev * pold[i];
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
  const bool with_x = PCG && d.do_xupd && a.defer_x;
  const double beta = d.beta;

  if (tid == 0) {
    mbar_init(mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // PCG pass A: persistent CTAs over blocks blockIdx.x, + gridDim.x, ... (of the list for a split pass
  // A); one grid reduction per CTA at the end, and the CTAs of an SM drift out of phase (one CTA's
  // staging overlaps another's arithmetic)
  const int nbl = a.blist ? a.nlist : (int)((K + E - 1) / E);
  double dot = 0.0;
  int it = 0;
  unsigned ph = 0;  // mbarrier phase (flips once per bulk-staged block)
#ifndef IPDG_TPB_PHASE
#define IPDG_TPB_PHASE 0  // measurement: clock64 phase durations of two CTAs printed at exit
#endif
  long long ph_acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, ph_last = 0;
#define TPB_MARK(k)                                                  \
  if constexpr (IPDG_TPB_PHASE != 0) {                               \
    const long long now_ = clock64();                                \
    if ((k) > 0) ph_acc[(k)] += now_ - ph_last;                      \
    ph_last = now_;                                                  \
  }
  auto block = [&](const int b) {
  TPB_MARK(0)
  if (it > 0) {  // the previous block's bulk store has read the rows before they are restaged
    if (tid == 0) bulk_wait_read();
    __syncthreads();
  }
  TPB_MARK(1)
  const int64_t e0 = (int64_t)b * E;
  const int Eb = (int)min((int64_t)E, K - e0);
  const int64_t g0 = e0 * NP;
  const int nrow = Eb * NP;
  // bulk copies of the block's rows when the byte count is a 16-byte multiple (every full block; the
  // caller's vectors are 16-byte aligned, checked at dispatch), else plain loads
  const bool bulk = ((nrow & 1) == 0);
  // per-element records of the own slots (R per thread: slots tid + r NTHR), loaded first so that their
  // latency overlaps the staging
  int sl[R];
  bool act[R];
  double Grr[R], Grs[R], Gss[R], Jv[R], tq3[R][3];
  short4 nb[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    sl[r] = tid + r * NTHR;
    act[r] = sl[r] < Eb;
    if (!act[r]) sl[r] = 0;  // idle slots compute on a valid row, never store
    const double4 gg = a.gG[e0 + sl[r]];
    Grr[r] = gg.x; Grs[r] = gg.y; Gss[r] = gg.z; Jv[r] = gg.w;
    nb[r] = a.nbt[e0 + sl[r]];
#pragma unroll
    for (int f = 0; f < 3; ++f) tq3[r][f] = a.tauF[(e0 + sl[r]) * 3 + f];
  }
  double* spo = sm + L::FT;              // PCG: p_{k-1} rows
  double* sx = sm + L::FT + E * NP;      // PCG: x rows
  if (bulk) {
    if (tid == 0) {
      const unsigned nb = (unsigned)nrow * 8u;
      mbar_expect_tx(mbar, nb * (1u + (with_p ? 1u : 0u) + (with_x ? 1u : 0u)));
      tma_load_1d(rows, U + g0, nb, mbar);
      if (with_p) tma_load_1d(spo, pold + g0, nb, mbar);
      if (with_x) tma_load_1d(sx, a.x + g0, nb, mbar);
    }
  } else {
    for (int q = tid; q < nrow; q += NTHR) {
      rows[q] = U[g0 + q];
      if (with_p) spo[q] = pold[g0 + q];
      if (with_x) sx[q] = a.x[g0 + q];
    }
  }

  TPB_MARK(2)
  // ---- ghost faces, while the bulk copies are in flight: value and trace of the outside neighbour on
  // the shared face, from its row in global memory (L2; PCG: p_k = z + beta p_{k-1}, the owner's FMA)
  // into the ghost-face records (their own region: no ordering against the staging)
  const int gf0 = a.gfoff[b], Gb = a.gfoff[b + 1] - gf0;
#ifndef IPDG_TPB_SKIP
#define IPDG_TPB_SKIP 0  // debug: 1 = no ghost pass, 2 = no volume, 4 = no face phase, 8 = no p/x formation (results wrong)
#endif
  for (int g = tid; g < ((IPDG_TPB_SKIP & 1) ? 0 : Gb); g += NTHR) {
    const int ent = a.gface[gf0 + g];
    const int64_t n = ent >> 2;
    const int fp = ent & 3;
    double un[NP];
    if (n >= K) {
      const double* h = a.halo_p + (n - K) * NP;
#pragma unroll
      for (int j = 0; j < NP; ++j) un[j] = h[j];
    } else {
      const double* src = U + n * NP;
      const double* po = pold + n * NP;
#pragma unroll
      for (int j = 0; j < NP; ++j) un[j] = with_p ? fma(beta, po[j], src[j]) : src[j];
    }
    const double4 gq = a.gG[n];
    double2* go = gft + g * NFP;
    if (fp == 0) ghost_face<N, 0>(un, gq, go);
    else if (fp == 1) ghost_face<N, 1>(un, gq, go);
    else ghost_face<N, 2>(un, gq, go);
  }

  TPB_MARK(3)
  if (bulk) { mbar_wait(mbar, ph); ph ^= 1u; }
  else __syncthreads();
  if (PCG && !(IPDG_TPB_SKIP & 8)) {  // p_k = z + beta p_{k-1} in place, p_k and the deferred x update x += alpha_{k-1} p_{k-1}
    const double alpha_prev = d.alpha_prev;
#pragma unroll 4
    for (int q = tid; q < nrow; q += NTHR) {
      const double po = with_p ? spo[q] : 0.0;
      const double v = with_p ? fma(beta, po, rows[q]) : rows[q];
      rows[q] = v;
      pnew[g0 + q] = v;
      if (with_x) a.x[g0 + q] = fma(alpha_prev, po, sx[q]);
    }
  }
  TPB_MARK(4)
  __syncthreads();  // p_k rows complete; staging consumed before the face records overwrite it
  TPB_MARK(5)

  // ---- own elements (R per thread: slots tid + r NTHR): volume, own face values and traces.  Outer
  // products: NP independent accumulators per element, every constant feeds R FMAs.
  auto row = [&](int r, int j) -> double { return rows[sl[r] * NP + j]; };
  double Au[R][NP];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int n = 0; n < NP; ++n) Au[r][n] = 0.0;
  if constexpr ((IPDG_TPB_SKIP & 2) != 0) {
  } else if constexpr (T::GRAD) {
    double wr[R][NP], ws[R][NP];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int i = 0; i < NP; ++i) wr[r][i] = ws[r][i] = 0.0;
#pragma unroll(T::UNR)
    for (int j = 0; j < NP; ++j) {  // [u_r | u_s] = [Dr u | Ds u]
      double uj[R];
#pragma unroll
      for (int r = 0; r < R; ++r) uj[r] = row(r, j);
#pragma unroll
      for (int i = 0; i < NP; ++i)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          wr[r][i] = fma(C[T::O_DRT + j * NP + i], uj[r], wr[r][i]);
          ws[r][i] = fma(C[T::O_DST + j * NP + i], uj[r], ws[r][i]);
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double2* fo = ft + sl[r] * TS;
#pragma unroll
      for (int i = 0; i < NP; ++i) {  // w = J G (u_r, u_s); face values and traces sJ n.grad u
        const double ur = wr[r][i], us = ws[r][i];
        wr[r][i] = Grr[r] * ur + Grs[r] * us;
        ws[r][i] = Grs[r] * ur + Gss[r] * us;
#pragma unroll
        for (int f = 0; f < 3; ++f)
#pragma unroll
          for (int k = 0; k < NFP; ++k)
            if (fmask_cf<N>(f, k) == i)
              fo[f * NFP + k] = make_double2(row(r, i), f == 0 ? -ws[r][i] : (f == 1 ? wr[r][i] + ws[r][i] : -wr[r][i]));
      }
    }
#pragma unroll
    for (int i = 0; i < NP; ++i) {  // Sr^T w_r + Ss^T w_s
#pragma unroll
      for (int n = 0; n < NP; ++n)
#pragma unroll
        for (int r = 0; r < R; ++r) Au[r][n] = fma(C[T::O_SR + i * NP + n], wr[r][i], Au[r][n]);
#pragma unroll
      for (int n = 0; n < NP; ++n)
#pragma unroll
        for (int r = 0; r < R; ++r) Au[r][n] = fma(C[T::O_SS + i * NP + n], ws[r][i], Au[r][n]);
    }
  } else {
  {  // own face values and traces sJ n.grad u
    double tf[R][NFP];
    face_trace<N, 0, R>(row, Grr, Grs, Gss, tf);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int k = 0; k < NFP; ++k) ft[sl[r] * TS + k] = make_double2(row(r, fmask_cf<N>(0, k)), tf[r][k]);
    face_trace<N, 1, R>(row, Grr, Grs, Gss, tf);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int k = 0; k < NFP; ++k) ft[sl[r] * TS + NFP + k] = make_double2(row(r, fmask_cf<N>(1, k)), tf[r][k]);
    face_trace<N, 2, R>(row, Grr, Grs, Gss, tf);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int k = 0; k < NFP; ++k) ft[sl[r] * TS + 2 * NFP + k] = make_double2(row(r, fmask_cf<N>(2, k)), tf[r][k]);
  }
  // volume: Au = Krr (J G_rr u) + Krs (J G_rs u) + Kss (J G_ss u) = Sr^T w_r + Ss^T w_s
#pragma unroll(T::UNR)
  for (int j = 0; j < NP; ++j) {
    double a0[R], a1[R], a2[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double uj = row(r, j);
      a0[r] = Grr[r] * uj; a1[r] = Grs[r] * uj; a2[r] = Gss[r] * uj;
    }
#pragma unroll
    for (int n = 0; n < NP; ++n)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        Au[r][n] = fma(C[T::O_KRR + j * NP + n], a0[r], Au[r][n]);
        Au[r][n] = fma(C[T::O_KRS + j * NP + n], a1[r], Au[r][n]);
        Au[r][n] = fma(C[T::O_KSS + j * NP + n], a2[r], Au[r][n]);
      }
  }
  }
  TPB_MARK(6)
  __syncthreads();  // face records of every slot (own and ghost) visible
  TPB_MARK(7)

  // ---- faces: jump, mirrored boundary traces (R7), flux, lift of the jump, face mass
#pragma unroll
  for (int f = 0; f < ((IPDG_TPB_SKIP & 4) ? 0 : 3); ++f) {
    double da[R][NFP], db[R][NFP], fg[R][NFP];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int fl = (nb[r].w >> (4 * f)) & 15;
      const int fp = fl & 3, bc = fl >> 2;
      const int slot = (f == 0) ? nb[r].x : (f == 1) ? nb[r].y : nb[r].z;
      const bool inner = (bc == 0);
      const double2* om = ft + sl[r] * TS + f * NFP;
      const double2* nbase = !inner ? om : (slot < E ? ft + slot * TS + fp * NFP : gft + (slot - E) * NFP);
      const bool flip = inner && ((f == 2) == (fp == 2));
      const double stau = tq3[r][f];
      // lift coefficients: c_r = 1/2 sJ n.grad r, c_s = 1/2 sJ n.grad s (k_geofacs) from J G:
      // face 0: (-G_rs, -G_ss)/2, face 1: (G_rr + G_rs, G_rs + G_ss)/2, face 2: (-G_rr, -G_rs)/2
      const double af = (f == 0) ? -0.5 * Gss[r] : (f == 1) ? 0.5 * (Grr[r] + 2.0 * Grs[r] + Gss[r]) : -0.5 * Grr[r];
      const double bf = (f == 0) ? -0.5 * Grs[r] : (f == 1) ? 0.5 * (Grs[r] + Gss[r]) : -0.5 * Grs[r];
#pragma unroll
      for (int k = 0; k < NFP; ++k) {
        const double2 m = om[k];
        const double2 p = nbase[flip ? NFP - 1 - k : k];
        const double delta = ((bc == 1) ? -p.x : p.x) - m.x;   // paper jump
        const double tq = (bc == 1) ? p.y : -p.y;               // sJ n-.grad u+
        fg[r][k] = -0.5 * (m.y + tq) - stau * delta;           // -sJ (n.{grad u} + tau delta)
        da[r][k] = af * delta;
        db[r][k] = bf * delta;
      }
    }
    if constexpr (!T::BIG) {
      // a_f T_f^T M1D delta (all nodes) + b_f D1D^T M1D delta + M1D (-sJ g) (face rows)
#pragma unroll
      for (int k = 0; k < NFP; ++k)
#pragma unroll
        for (int m = 0; m < NFP; ++m)
#pragma unroll
          for (int r = 0; r < R; ++r) {
            double& o = Au[r][fmask_cf<N>(f, m)];
            o = fma(C[T::O_QT + k * NFP + m], db[r][k], o);
            o = fma(C[T::O_M1D + k * NFP + m], fg[r][k], o);
          }
#pragma unroll(T::FULLF ? NFP : 1)
      for (int k = 0; k < NFP; ++k)
#pragma unroll
        for (int n = 0; n < NP; ++n)
#pragma unroll
          for (int r = 0; r < R; ++r) Au[r][n] = fma(C[T::O_PT + (f * NFP + k) * NP + n], da[r][k], Au[r][n]);
    } else {
      // md = M1D delta; a_f T_f^T md (all nodes) + b_f D1D^T md + M1D (-sJ g) (face rows)
      double md[R][NFP], mb[R][NFP];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int m = 0; m < NFP; ++m) {
          double v = 0.0, w = 0.0;
#pragma unroll
          for (int k = 0; k < NFP; ++k) {
            v = fma(C[T::O_M1D + m * NFP + k], da[r][k], v);
            w = fma(C[T::O_M1D + m * NFP + k], db[r][k], w);
          }
          md[r][m] = v;
          mb[r][m] = w;
        }
#pragma unroll
      for (int k = 0; k < NFP; ++k)
#pragma unroll
        for (int m = 0; m < NFP; ++m)
#pragma unroll
          for (int r = 0; r < R; ++r) {
            double& o = Au[r][fmask_cf<N>(f, m)];
            o = fma(C[T::O_D1DT + m * NFP + k], mb[r][k], o);
            o = fma(C[T::O_M1D + k * NFP + m], fg[r][k], o);
          }
#pragma unroll 1
      for (int k = 0; k < NFP; ++k)
#pragma unroll
        for (int n = 0; n < NP; ++n)
#pragma unroll
          for (int r = 0; r < R; ++r) Au[r][n] = fma(C[T::O_TN + (f * NFP + k) * NP + n], md[r][k], Au[r][n]);
    }
  }
  if constexpr (LAM && T::HAS_LAM) {  // lambda J M u, own rows from shared memory
#pragma unroll(T::UNR)
    for (int j = 0; j < NP; ++j) {
      double uj[R];
#pragma unroll
      for (int r = 0; r < R; ++r) uj[r] = a.lambda * Jv[r] * row(r, j);
#pragma unroll
      for (int n = 0; n < NP; ++n)
#pragma unroll
        for (int r = 0; r < R; ++r) Au[r][n] = fma(C[T::O_M + j * NP + n], uj[r], Au[r][n]);
    }
  }
  // Au in place over the own rows (phase 2 reads only the face records, never another thread's row)
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (act[r]) {
      double* wo = rows + sl[r] * NP;
#pragma unroll
      for (int n = 0; n < NP; ++n) {
        if (PCG) dot = fma(wo[n], Au[r][n], dot);
        wo[n] = Au[r][n];
      }
    }
  if (bulk) fence_proxy_async();  // generic-proxy writes -> visible to the bulk copy
  __syncthreads();
  if (bulk) {
    if (tid == 0) bulk_store(a.Au + g0, rows, (unsigned)nrow * 8u);
  } else {
    for (int q = tid; q < nrow; q += NTHR) a.Au[g0 + q] = rows[q];
  }
  TPB_MARK(8)
  ++it;
  };  // block
  // PCG pass A: persistent CTAs (grid = resident CTAs x SMs, IPDG_TPB_PERSIST); Ax: one CTA per block
  // (the loop costs the Ax instance registers and spills, measured slower)
  if constexpr (PCG) {
    for (int bi = blockIdx.x; bi < nbl; bi += gridDim.x) block(a.blist ? a.blist[bi] : bi);
  } else {
    block(a.blist ? a.blist[blockIdx.x] : (int)blockIdx.x);
  }
  if (PCG) {
    double v[1] = {dot}, out[1];
    if (grid_reduce<1>(v, red, a.partials, a.counter, out)) {
      PcgState* st = a.st;
      if (a.red_part == 1) st->red_A_part = out[0];
      else st->red_A = (a.red_part == 2) ? st->red_A_part + out[0] : out[0];
      st->rho_hist[(d.k - 1) & 3] = d.rhoB;
      if (d.first) st->bb = d.bbv;
    }
  }
  if (tid == 0) bulk_wait_read();  // the last bulk store has read the rows before the CTA exits
  if constexpr (IPDG_TPB_PHASE != 0) {
    if (blockIdx.x < 3 && (tid == 0 || tid == 96))
      printf("TPB_PHASE mode=%d cta=%d tid=%d blocks=%d wait=%lld rec=%lld ghost=%lld mbar_form=%lld bar1=%lld vol=%lld bar2=%lld face_store=%lld\n",
             MODE, (int)blockIdx.x, tid, it, ph_acc[1], ph_acc[2], ph_acc[3], ph_acc[4], ph_acc[5], ph_acc[6], ph_acc[7], ph_acc[8]);
  }
}

}  // namespace ipdg
