// Software-pipelined fused SIPDG kernel (variant 4).  Paper: arXiv:1801.00246; formulation in
// kernels.cuh, phase structure as k_sipdg (sipdg_kernels.cuh):
//   P1  [u_r | u_s] = u [Dr^T | Ds^T] on DMMA for own + ghost tiles      (Alg. AxG)
//   P2  jump, mirrored boundary traces, central flux + penalty per own face node
//                                                                          (Alg. AxKernel)
//   P3  Au = [w_r | w_s | face block] x [Sr; Ss; LIFT^T Sr; LIFT^T Ss; E^T] on DMMA (+ lambda J M u)
// What differs from k_sipdg: the element data of block b+1 (own rows by TMA bulk copies, ghost rows
// and geometry by cp.async) streams into a staging area while block b computes, so the HBM/L2 load
// latency of a block overlaps the previous block's DMMA work instead of stalling every CTA at the top
// of each block (the P0 phase took 37 % of k_sipdg's PCG pass A, profiles/r01_phase_timing_fused_N4.txt).
// At the top of a block the staged rows are consumed into the working rows `us` (PCG pass A forms
// p_k = z + beta p_{k-1} there, writes p_k and the deferred x update), which frees the staging area
// for the next block.  Only the face traces sJ n.grad u (3 Nfp per slot) are kept for the flux,
// not the full w_r | w_s rows, which pays for the staging area in shared memory.
#pragma once
#include "sipdg_kernels.cuh"
#include "sipdg_split.cuh"

namespace ipdg {

template <int N>
struct TrPipe {
  using T = Tr<N>;
  static constexpr int TS = (T::NF3 + 1) | 1;   // trace row stride (odd: gathers spread over banks); column NF3 = junk
  static constexpr int OSTR = T::E * T::NP + 2;  // own staging array stride (TMA head alignment pad)
};

struct PipeLayout {
  int tabG, tabM, tabL, iaux, ncode, meta, us, trc, geo, fg, nb, gid, stg, mbar, total;  // offsets in doubles
  template <int N>
  __host__ __device__ static PipeLayout make(int gmax, bool lam, bool pcg) {
    using T = Tr<N>;
    using P = TrPipe<N>;
    PipeLayout L;
    const int gm8 = (gmax + 7) / 8 * 8;
    const int slots = T::E + gm8;
    int o = 0;
    L.tabG = o; o += T::TAB_G;
    L.tabM = o; o += T::TAB_M;
    L.tabL = o; o += lam ? T::TAB_L : 0;
    L.iaux = o; o += (6 * T::NFP + 1) / 2;   // ints: nidx[f'][flip][k]
    L.ncode = o;
    L.meta = o; o += 8;                       // ints: 4 x (e0, e1, g0, g1) block metadata ring
    o = (o + 1) & ~1;
    L.us = o; o += slots * T::SU;
    L.trc = o; o += slots * P::TS;
    o = (o + 1) & ~1;
    L.geo = o; o += 2 * slots * T::SG;        // double-buffered: rx sx ry sy J - - -
    L.fg = o; o += 9 * T::FGS;
    L.nb = o; o += 2 * T::E;                  // short4, double-buffered
    L.gid = o; o += gm8;                      // 2 x gm8 ints
    o = (o + 1) & ~1;
    L.stg = o; o += (pcg ? 3 : 1) * P::OSTR + (pcg ? 2 : 1) * gm8 * T::NP;
    o = (o + 1) & ~1;
    L.mbar = o; o += 1;
    L.total = o;
    return L;
  }
};

// trace columns of reference node i (row-by-row node order, refops.cpp): bits 5f..5f+4 = the column
// f*Nfp + k of the trace row when Fmask[f][k] = i, else the junk column 3 Nfp (branch-free stores)
template <int N>
__host__ __device__ inline int node_trace_cols(int i) {
  constexpr int NFP = N + 1, JUNK = 3 * (N + 1);
  int j = 0, off = 0;
  while (j <= N && off + (N + 1 - j) <= i) { off += N + 1 - j; ++j; }
  if (j > N) return JUNK | (JUNK << 5) | (JUNK << 10);
  const int m = i - off;
  const int c0 = (j == 0) ? m : JUNK;
  const int c1 = (m == N - j) ? NFP + j : JUNK;
  const int c2 = (m == 0) ? 2 * NFP + j : JUNK;
  return c0 | (c1 << 5) | (c2 << 10);
}

template <int N, int MODE, bool LAM>
__global__ void __launch_bounds__(Tr<N>::W * 32, Tr<N>::MINB) k_pipe(AxArgs a, int gmax) {
  using T = Tr<N>;
  using P = TrPipe<N>;
  constexpr int NP = T::NP, NFP = T::NFP, NT = T::NT, NPN = T::NPN, SU = T::SU, SG = T::SG, TS = P::TS;
  constexpr int W = T::W, E = T::E, KCG = T::KCG, KCW = T::KCW, KCM = T::KCM, OSTR = P::OSTR;
  constexpr int NTHR = W * 32;
  constexpr bool PCG = (MODE == MODE_PCG_A);
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[32 * 3];
  const PipeLayout L = PipeLayout::make<N>(gmax, LAM, PCG);
  const int gm8 = (gmax + 7) / 8 * 8;
  const int slots = E + gm8;
  double* tabG = sm + L.tabG;
  double* tabM = sm + L.tabM;
  double* tabL = sm + L.tabL;
  int* nidx = reinterpret_cast<int*>(sm + L.iaux);
  int* meta = reinterpret_cast<int*>(sm + L.meta);
  double* us = sm + L.us;
  double* trc = sm + L.trc;
  double* geo0 = sm + L.geo;
  double* fgs = sm + L.fg;
  short4* nbs0 = reinterpret_cast<short4*>(sm + L.nb);
  int* gids0 = reinterpret_cast<int*>(sm + L.gid);
  double* stg = sm + L.stg;
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(sm + L.mbar);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t K = a.K;
  const int G = gridDim.x;

  PcgDecision d;
  double dot = 0.0;
  double* pnew = nullptr;
  const double* pold = nullptr;
  const double* U = a.u;
  if (PCG) {
    PcgState* st = a.st;
    if (st->stop_iter >= 0) return;  // stopped by an earlier launch
    d = pcg_decide(st);
    pnew = (d.k & 1) ? a.p_odd : a.p_even;
    pold = (d.k & 1) ? a.p_even : a.p_odd;
    U = a.z;
    if (d.stop) {
      const int64_t n = K * NP;
      for (int64_t i = blockIdx.x * (int64_t)NTHR + tid; i < n; i += (int64_t)G * NTHR) {
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
  const bool with_p = PCG && !d.first;   // p_{k-1} staged
  const bool with_x = PCG && d.do_xupd;  // x staged for the deferred update

  // ---- once per CTA: operator tables, index tables, zero padding, metadata of the first blocks
  {
    const double* src = a.tables;
    constexpr int ntab = T::TAB_G + T::TAB_M + (LAM ? T::TAB_L : 0);  // multiple of 32 doubles
    for (int i = 2 * tid; i < ntab; i += 2 * NTHR) cp_async16(sm + i, src + i);
    for (int q = tid; q < 6 * NFP; q += NTHR) {  // nidx[fp][flip][k] = Fmask[fp][flip ? Nfp-1-k : k]
      const int fp = q / (2 * NFP), fl = (q / NFP) & 1, kk = q % NFP;
      nidx[q] = fmask_cf<N>(fp, fl ? NFP - 1 - kk : kk);
    }
    for (int i = tid; i < slots * SU; i += NTHR) us[i] = 0.0;  // padding columns stay zero
    if (tid < 12) {  // metadata of this CTA's blocks 0, 1, 2 -> ring slots 0, 1, 2
      const int j = tid >> 2, w = tid & 3;
      const int b = blockIdx.x + j * G;
      int v = 0;
      if (b < a.nblocks) v = (w < 2) ? a.boff[b + w] : a.goff[b + w - 2];
      meta[4 * j + w] = v;
    }
    if (tid == 0) {
      mbar_init(mbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (blockIdx.x < a.nblocks) {  // ghost ids of block 0 (plain loads, once)
      const int g0 = meta[2], g1 = meta[3];
      for (int g = tid; g < g1 - g0; g += NTHR) gids0[g] = a.gid[g0 + g];
    }
    __syncthreads();
  }

  // ---- issue the loads of one block into the staging area (own rows by TMA when possible)
  int tma_phase = 0;
  auto issue = [&](int gpar, const int* mt, const int* gl, int& shift, bool& tma) {
    const int64_t e0 = mt[0];
    const int Eb = mt[1] - mt[0], Gb = mt[3] - mt[2];
    double* gb = geo0 + gpar * slots * SG;
    short4* nb = nbs0 + gpar * E;
    for (int q = tid; q < 2 * (Eb + Gb); q += NTHR) {  // raw geometry r_x s_x r_y s_y (2 x 16 B)
      const int s = q >> 1, h = q & 1;
      const int slot = s < Eb ? s : E + (s - Eb);
      const int64_t el = s < Eb ? e0 + s : (int64_t)gl[s - Eb];
      cp_async16(gb + slot * SG + 2 * h, reinterpret_cast<const double*>(a.geo + el) + 2 * h);
    }
    for (int e = tid; e < Eb; e += NTHR) cp_async8(nb + e, a.nbr + e0 + e);
    // own rows: one contiguous range per vector -> TMA bulk copy (16-byte aligned: the copy starts
    // one double early when the range starts on an odd double; the tail block falls back to cp.async)
    const int64_t g0 = e0 * NP;
    shift = (int)(g0 & 1);
    const int64_t gbase = g0 - shift;
    const unsigned nbytes = (unsigned)(((Eb * NP + shift) * 8 + 15) & ~15);
    tma = (gbase + nbytes / 8 <= K * NP);
    double* s0 = stg;
    double* s1 = stg + OSTR;
    double* s2 = stg + 2 * OSTR;
    if (tma) {
      if (tid == 0) {
        const unsigned tot = nbytes * (1u + (with_p ? 1u : 0u) + (with_x ? 1u : 0u));
        mbar_expect_tx(mbar, tot);
        tma_load_1d(s0, U + gbase, nbytes, mbar);
        if (with_p) tma_load_1d(s1, pold + gbase, nbytes, mbar);
        if (with_x) tma_load_1d(s2, a.x + gbase, nbytes, mbar);
      }
    } else {
      shift = 0;
      for (int q = tid; q < Eb * NP; q += NTHR) {
        cp_async8(s0 + q, U + g0 + q);
        if (with_p) cp_async8(s1 + q, pold + g0 + q);
        if (with_x) cp_async8(s2 + q, a.x + g0 + q);
      }
    }
    double* gz = stg + (PCG ? 3 : 1) * OSTR;
    double* gp = gz + gm8 * NP;
    for (int q = tid; q < Gb * NP; q += NTHR) {
      const int g = q / NP, i = q - g * NP;
      const int ge = gl[g];
      if (ge >= K) {
        cp_async8(gz + q, a.halo_p + (int64_t)(ge - K) * NP + i);
      } else {
        cp_async8(gz + q, U + (int64_t)ge * NP + i);
        if (with_p) cp_async8(gp + q, pold + (int64_t)ge * NP + i);
      }
    }
  };

  // trace columns of this lane's C-fragment nodes 8 nt + 2 (lane & 3) + h
  int tcol[2 * NT];
#pragma unroll
  for (int q = 0; q < 2 * NT; ++q) tcol[q] = node_trace_cols<N>(8 * (q >> 1) + 2 * (lane & 3) + (q & 1));
  // per-lane face-node items for P2 (4 lanes per element): fk = 4q + (lane & 3) -> (f, k, node)
  int itab[T::NQ];
#pragma unroll
  for (int q = 0; q < T::NQ; ++q) {
    const int fk = 4 * q + (lane & 3);
    const int f = fk / NFP, kk = fk - f * NFP;
    itab[q] = (fk < T::NF3) ? ((f << 24) | (kk << 16) | fmask_cf<N>(f, kk))
                            : ((2 << 24) | (N << 16) | fmask_cf<N>(2, N));  // pad: any finite value (zero B rows)
  }

  int cur_shift = 0, nxt_shift = 0;
  bool cur_tma = false, nxt_tma = false;
  if (blockIdx.x < a.nblocks) {
    issue(0, meta, gids0, cur_shift, cur_tma);
    const int b1 = blockIdx.x + G;
    if (b1 < a.nblocks) {  // ghost ids of block 1 -> gids[1]
      const int g0 = meta[4 + 2], g1 = meta[4 + 3];
      for (int g = tid; g < g1 - g0; g += NTHR) cp_async4(gids0 + gm8 + g, a.gid + g0 + g);
    }
  }
  cp_async_commit();

  double wr[NT][2], ws[NT][2];
  int it = 0;
  for (int b = blockIdx.x; b < a.nblocks; b += G, ++it) {
    const int par = it & 1;
    const int* mt = meta + 4 * (it & 3);
    const int64_t e0 = mt[0];
    const int Eb = mt[1] - mt[0], Gb = mt[3] - mt[2];
    int* gids = gids0 + par * gm8;
    double* geos = geo0 + par * slots * SG;
    short4* nbs = nbs0 + par * E;
    // ---- wait for this block's staged data (issued one block earlier)
    cp_async_wait_all();
    if (cur_tma) {
      mbar_wait(mbar, tma_phase);
      tma_phase ^= 1;
    }
    __syncthreads();
    // ---- consume: staged rows -> working rows (PCG: p_k = z + beta p_{k-1}, deferred x update)
    {
      const double* s0 = stg + cur_shift;
      const double* s1 = stg + OSTR + cur_shift;
      const double* s2 = stg + 2 * OSTR + cur_shift;
      const double* gz = stg + (PCG ? 3 : 1) * OSTR;
      const double* gp = gz + gm8 * NP;
      for (int q = tid; q < Eb * NP; q += NTHR) {
        const int e = q / NP, i = q - e * NP;
        double v = s0[q];
        if (PCG) {
          const double po = with_p ? s1[q] : 0.0;
          v += d.beta * po;
          const int64_t g = e0 * NP + q;
          pnew[g] = v;
          if (with_x) a.x[g] = s2[q] + d.alpha_prev * po;
        }
        us[e * SU + i] = v;
      }
      for (int q = tid; q < Gb * NP; q += NTHR) {
        const int g = q / NP, i = q - g * NP;
        double v = gz[q];
        if (with_p && gids[g] < K) v += d.beta * gp[q];
        us[(E + g) * SU + i] = v;
      }
    }
    // ---- per-slot geometry, one thread per slot (not per lane of the DMMA tiles):
    // J G^T G entries for the chain rule; own slots also the per-face lift coefficients and sJ tau
    if (tid < Eb + Gb) {
      const int slot = tid < Eb ? tid : E + (tid - Eb);
      double* gq = geos + slot * SG;
      const double rx = gq[0], sx = gq[1], ry = gq[2], sy = gq[3];
      const double det = rx * sy - sx * ry;  // = 1/J
      const double J = 1.0 / det;
      gq[4] = J * (rx * rx + ry * ry);  // J G_rr
      gq[5] = J * (rx * sx + ry * sy);  // J G_rs
      gq[6] = J * (sx * sx + sy * sy);  // J G_ss
      gq[7] = J;
      if (tid < Eb) {
        const short4 nb = nbs[slot];
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          const double gx = (f == 0) ? -sx : (f == 1) ? rx + sx : -rx;  // outward: -grad s, grad r+s, -grad r
          const double gy = (f == 0) ? -sy : (f == 1) ? ry + sy : -ry;
          const double sJ = J * sqrt(gx * gx + gy * gy);                 // edge length / 2 (R6)
          const int bc = (nb.w >> (4 * f + 2)) & 3;
          double detp = 0.0;                                             // neighbour det G (= 1/J+) on interior faces
          if (bc == 0) {
            const double* gn = geos + ((f == 0) ? nb.x : (f == 1) ? nb.y : nb.z) * SG;
            detp = gn[0] * gn[3] - gn[1] * gn[2];
          }
          double* fq = fgs + 3 * f * T::FGS + slot;
          fq[0] = 0.5 * J * (rx * gx + ry * gy);                          // 1/2 sJ (n . grad r)
          fq[T::FGS] = 0.5 * J * (sx * gx + sy * gy);                     // 1/2 sJ (n . grad s)
          fq[2 * T::FGS] = sJ * a.tau_c * sJ * fmax(det, detp);           // sJ tau, Eq. Ch2.PenaltyParameter (1/h = sJ/J)
        }
      }
    }
    {  // metadata of block b + 3G -> ring slot (it + 3) & 3 (read two iterations later)
      const int b3 = b + 3 * G;
      if (tid < 4 && b3 < a.nblocks) {
        int* m3 = meta + 4 * ((it + 3) & 3);
        if (tid < 2) cp_async4(m3 + tid, a.boff + b3 + tid);
        else cp_async4(m3 + tid, a.goff + b3 + tid - 2);
      }
    }
    __syncthreads();  // staging area and gids[par] free
    // ---- issue block b + G (staging) and the ghost ids of block b + 2G (gids[par])
    {
      const int b1 = b + G, b2 = b + 2 * G;
      if (b1 < a.nblocks) issue(par ^ 1, meta + 4 * ((it + 1) & 3), gids0 + (par ^ 1) * gm8, nxt_shift, nxt_tma);
      else nxt_tma = false;
      if (b2 < a.nblocks) {
        const int* m2 = meta + 4 * ((it + 2) & 3);
        const int g0 = m2[2], g1 = m2[3];
        for (int g = tid; g < g1 - g0; g += NTHR) cp_async4(gids + g, a.gid + g0 + g);
      }
      cp_async_commit();
    }

    // ---- P1: reference gradient on DMMA; face traces to smem; w_r / w_s kept in registers (own)
    const int ntiles = W + (Gb + 7) / 8;
    for (int t = warp; t < ntiles; t += W) {
      const bool own = t < W;
      const int sbase = own ? 8 * t : E + 8 * (t - W);
      if (own && sbase >= Eb) continue;
      double acc[2 * NT][2];
#pragma unroll
      for (int q = 0; q < 2 * NT; ++q) acc[q][0] = acc[q][1] = 0.0;
      const int srow = sbase + (lane >> 2);
      const double* urow = us + srow * SU + (lane & 3);
#pragma unroll
      for (int kc = 0; kc < KCG; ++kc) {
        const double av = urow[4 * kc];
        const double* bt = tabG + kc * 2 * NT * 32 + lane;
#pragma unroll
        for (int q = 0; q < 2 * NT; ++q) dmma(acc[q][0], acc[q][1], av, bt[q * 32]);
      }
      // w_r = J (G_rr u_r + G_rs u_s), w_s = J (G_rs u_r + G_ss u_s); the scaled normal derivatives
      // sJ n.grad u on faces 0, 1, 2 are -w_s, w_r + w_s, -w_r (J g_f.grad u, g_f = -grad s,
      // grad r + grad s, -grad r)
      const double* gq = geos + srow * SG;
      const double Grr = gq[4], Grs = gq[5], Gss = gq[6];
      double* trow = trc + srow * TS;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double ur0 = acc[nt][0], ur1 = acc[nt][1], us0 = acc[NT + nt][0], us1 = acc[NT + nt][1];
        const double r0 = Grr * ur0 + Grs * us0, r1 = Grr * ur1 + Grs * us1;
        const double s0 = Grs * ur0 + Gss * us0, s1 = Grs * ur1 + Gss * us1;
        // traces stored as -sJ n.grad u: w_s, -(w_r + w_s), w_r on faces 0, 1, 2 (junk column if the
        // node is not on the face)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = tcol[2 * nt + h];
          const double wrv = h ? r1 : r0, wsv = h ? s1 : s0;
          trow[c & 31] = wsv;
          trow[(c >> 5) & 31] = -(wrv + wsv);
          trow[(c >> 10) & 31] = wrv;
        }
        if (own) {
          wr[nt][0] = r0;
          wr[nt][1] = r1;
          ws[nt][0] = s0;
          ws[nt][1] = s1;
        }
      }
    }
    // ---- P3 volume part per warp on its own tile, straight from registers (no barrier needed: warps
    // with fewer P1 tiles start here while the others finish theirs)
    const int e = 8 * warp + (lane >> 2);
    double C[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) C[nt][0] = C[nt][1] = 0.0;
    if (8 * warp < Eb) {
#pragma unroll
      for (int c = 0; c < 2 * NT; ++c) {
        const double av = wr[c >> 1][c & 1];
        const double* bt = tabM + c * NT * 32 + lane;
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(C[j][0], C[j][1], av, bt[j * 32]);
      }
#pragma unroll
      for (int c = 0; c < 2 * NT; ++c) {
        const double av = ws[c >> 1][c & 1];
        const double* bt = tabM + (2 * NT + c) * NT * 32 + lane;
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(C[j][0], C[j][1], av, bt[j * 32]);
      }
    }
    __syncthreads();  // traces of every slot written

    // ---- P2 + P3 face part per warp on its own tile
    if (8 * warp < Eb) {
      {
        const int ec = e < Eb ? e : 8 * warp;  // rows past the block end compute on a valid slot, never stored
        const short4 nb = nbs[ec];
        const double* uo = us + ec * SU;
        const double* to = trc + ec * TS;
        const double* fq0 = fgs + ec;
#pragma unroll
        for (int q = 0; q < T::NQ; ++q) {
          const int itq = itab[q];
          const int f = itq >> 24, kk = (itq >> 16) & 255, i = itq & 65535;
          const int fl = (nb.w >> (4 * f)) & 15;
          const int fp = fl & 3, bc = fl >> 2;
          const int slot = (f == 0) ? nb.x : (f == 1) ? nb.y : nb.z;
          const double* fq = fq0 + 3 * f * T::FGS;
          // boundary faces read the element's own trace and mirror it (R7):
          // Dirichlet u+ = -u-, grad u+ = grad u-;  Neumann u+ = u-, grad u+ = -grad u-
          const bool inner = (bc == 0);
          const int flip = inner && ((f == 2) == (fp == 2));
          const int ps = inner ? slot : ec;
          const int kq = flip ? NFP - 1 - kk : kk;
          const int tpi = inner ? fp * NFP + kq : f * NFP + kk;
          const int ip = inner ? nidx[(2 * fp + flip) * NFP + kk] : i;
          const double um = uo[i], upr = us[ps * SU + ip];
          const double tm = to[f * NFP + kk];     // -sJ n-.grad u-
          const double tp = trc[ps * TS + tpi];   // -sJ n+.grad u+ (the neighbour's own normal)
          const double delta = ((bc == 1) ? -upr : upr) - um;     // paper jump
          const double far = fq[0] * delta;                       // 1/2 sJ (n.grad r) delta
          const double fas = fq[T::FGS] * delta;                  // 1/2 sJ (n.grad s) delta
          // -sJ (n-.{grad u} + tau delta); n-.grad u+ = -n+.grad u+ inside, = n-.grad u- mirrored on Dirichlet
          const double hp = (bc == 1) ? 0.5 : -0.5;
          const double fag = fma(0.5, tm, fma(hp, tp, -fq[2 * T::FGS] * delta));
          const double* b0 = tabM + (KCW + q) * NT * 32 + lane;
          const double* b1 = tabM + (KCW + T::NQ + q) * NT * 32 + lane;
          const double* b2 = tabM + (KCW + 2 * T::NQ + q) * NT * 32 + lane;
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            dmma(C[j][0], C[j][1], far, b0[j * 32]);
            dmma(C[j][0], C[j][1], fas, b1[j * 32]);
            dmma(C[j][0], C[j][1], fag, b2[j * 32]);
          }
        }
      }
      if (LAM) {
        const double lj = a.lambda * geos[e * SG + 7];
        const double* urow = us + e * SU + (lane & 3);
#pragma unroll
        for (int kc = 0; kc < KCM; ++kc) {
          const double av = lj * urow[4 * kc];
          const double* bt = tabL + kc * NT * 32 + lane;
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma(C[j][0], C[j][1], av, bt[j * 32]);
        }
      }
      if (e < Eb) {
        const int64_t base = (e0 + e) * NP;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int i = 8 * nt + 2 * (lane & 3) + h;
            if (i < NP) {
              a.Au[base + i] = C[nt][h];
              if (PCG) dot += us[e * SU + i] * C[nt][h];
            }
          }
      }
    }
    cur_shift = nxt_shift;
    cur_tma = nxt_tma;
  }
  cp_async_wait_all();
  if (PCG) {
    double v[1] = {dot}, out[1];
    if (grid_reduce<1>(v, red, a.partials, a.counter, out)) {
      PcgState* st = a.st;
      st->red_A = out[0];
      st->rho_hist[(d.k - 1) & 3] = d.rhoB;
      if (d.first) st->bb = d.bbv;
    }
  }
}

}  // namespace ipdg
