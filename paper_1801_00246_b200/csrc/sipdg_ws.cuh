// Warp-specialised pipelined fused SIPDG kernel (variant 6, k_ws).  Paper: arXiv:1801.00246;
// formulation in kernels.cuh, phases as k_pipe (sipdg_pipe.cuh):
//   P1  [u_r | u_s] = u [Dr^T | Ds^T] on DMMA for own + ghost tiles      (Alg. AxG)
//   P2  jump, mirrored boundary traces, central flux + penalty per own face node
//                                                                          (Alg. AxKernel)
//   P3  Au = [w_r | w_s | face block] x [Sr; Ss; LIFT^T Sr; LIFT^T Ss; E^T] on DMMA (+ lambda J M u)
// What differs from k_pipe (measured there: latency / barrier bound, ~20 % of the time in the load
// issue, ~15 % in the p / x pass, ~30 warp instructions per element decoding face-node gathers):
//  * One producer warp per CTA does all the non-tensor work of a block ahead of the compute warps:
//    it issues the loads of block b+1 (own rows, records by TMA bulk copies; ghost rows by cp.async
//    tracked on the same mbarrier), decodes the neighbour slots into one gather descriptor per own face,
//    and in PCG pass A forms p_k = z + beta p_{k-1} in place (own and ghost rows), writes p_k and the
//    deferred x += alpha_{k-1} p_{k-1} of the own rows -- so the compute warps see an Ax on staged rows.
//    full / ready / empty mbarriers per stage; no CTA-wide barrier in the block loop.
//  * Own and ghost rows live in one slot-indexed array (stride N_p): operand reads are branch-free.
//  * P1 also stores u at the face nodes beside the face traces -sJ n.grad u, so P2 reads both sides of
//    every face node from the trace rows at offsets given by the descriptor (no node-index decode).
//  * Each compute warp owns TT element tiles (TT = 2: every operator fragment loaded from shared memory
//    feeds two DMMAs, twice the independent accumulator chains per warp).
#pragma once
#include "sipdg_pipe.cuh"

namespace ipdg {

template <int N>
struct TrW {
  using T = Tr<N>;
  static constexpr int WC = 8;               // compute warps
  static constexpr int TT = 1;               // own 8-element tiles per compute warp
  static constexpr int E = 8 * TT * WC;      // own elements per block (= Tr<N>::E: same block schedule)
  static constexpr int NTHR = (WC + 1) * 32; // + one producer warp
  static constexpr int UO = T::NF3 + 4;      // trace row: [0, NF3) -sJ n.grad u | 4 junk | [UO, UO+NF3) u | 4 junk
  static constexpr int TS = (2 * UO) | 1;
  static_assert(E == T::E, "k_ws uses the k_pipe block schedule");
};

struct WsLayout {
  // offsets in doubles
  int tabG, tabM, tabL, iaux, trc, mbar, pold, stg, sz;
  int o_rows, o_gG, o_gF, o_fd, o_meta;  // within one stage
  template <int N>
  __host__ __device__ static WsLayout make(int gmax, bool lam, bool pcg) {
    using T = Tr<N>;
    using W = TrW<N>;
    WsLayout L;
    const int gm8 = (gmax + 7) / 8 * 8;
    const int slots = W::E + gm8;
    int o = 0;
    L.tabG = o; o += T::TAB_G;
    L.tabM = o; o += T::TAB_M;
    L.tabL = o; o += lam ? T::TAB_L : 0;
    L.iaux = o; o += 0;
    o = (o + 1) & ~1;
    L.trc = o; o += slots * W::TS;
    o = (o + 1) & ~1;
    L.mbar = o; o += 6;                        // full[2], ready[2], empty[2]
    L.pold = o; o += pcg ? slots * T::NP + 2 : 0;  // p_{k-1} rows of the block being formed (producer only)
    o = (o + 1) & ~1;
    int q = 0;
    L.o_rows = q; q += slots * T::NP + 2;      // operand rows (+2: TMA alignment shift)
    q = (q + 1) & ~1;
    L.o_gG = q; q += slots * 4;
    L.o_gF = q; q += W::E * kGF;
    L.o_fd = q; q += 3 * W::E;                 // int2 per own face: neighbour trace-row base, flags
    L.o_meta = q; q += 2;                      // ints: e0, Eb, Gb
    q = (q + 1) & ~1;
    L.sz = q;
    L.stg = o;
    return L;
  }
  __host__ __device__ int total() const { return stg + 2 * sz; }
};

__device__ __forceinline__ void cp_async_mbar_arrive_noinc(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

template <int N, int MODE, bool LAM>
__global__ void __launch_bounds__(TrW<N>::NTHR, 2) k_ws(AxArgs a, int gmax) {
  using T = Tr<N>;
  using W = TrW<N>;
  constexpr int NP = T::NP, NFP = T::NFP, NT = T::NT, TS = W::TS, UO = W::UO, GF = kGF;
  constexpr int WC = W::WC, TT = W::TT, E = W::E, KCG = T::KCG, KCW = T::KCW, KCM = T::KCM, NQ = T::NQ;
  constexpr int NTHR = W::NTHR, NCT = WC * 32;
  constexpr bool PCG = (MODE == MODE_PCG_A);
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[32 * 3];
  const WsLayout L = WsLayout::make<N>(gmax, LAM, PCG);
  double* tabG = sm + L.tabG;
  double* tabM = sm + L.tabM;
  double* tabL = sm + L.tabL;
  double* trc = sm + L.trc;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sm + L.mbar);
  unsigned long long* ready = full + 2;
  unsigned long long* empty = full + 4;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t K = a.K;
  const int G = gridDim.x;
  const int nbl = a.blist ? a.nlist : a.nblocks;

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
  const bool with_p = PCG && !d.first;                // p_{k-1} staged: p_k = z + beta p_{k-1}
  const bool with_x = PCG && d.do_xupd;               // deferred x += alpha_{k-1} p_{k-1}
  const double beta = with_p ? d.beta : 0.0, alpha_prev = d.alpha_prev;

  // ---- once per CTA: operator tables, zeroed stages (padding rows stay finite), barriers
  {
    constexpr int ntab = T::TAB_G + T::TAB_M + (LAM ? T::TAB_L : 0);
    for (int i = 2 * tid; i < ntab; i += 2 * NTHR) cp_async16(sm + i, a.tables + i);
    cp_async_commit();
    for (int i = tid; i < L.total() - L.trc; i += NTHR) sm[L.trc + i] = 0.0;
    __syncthreads();
    if (tid == 0) {
      for (int s = 0; s < 2; ++s) {
        mbar_init(full + s, 33);   // producer lane 0 (arrive.expect_tx) + 32 cp.async arrivals
        mbar_init(ready + s, 1);   // producer lane 0 once p_k is formed (PCG)
        mbar_init(empty + s, WC);  // one arrival per compute warp
      }
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    cp_async_wait_all();
    __syncthreads();
  }

  if (warp == WC) {
    // ================================================================ producer warp
    int it = 0;
    int nb_e0 = 0, nb_e1 = 0, nb_g0 = 0, nb_g1 = 0;
    if (blockIdx.x < nbl) {
      const int bi = a.blist ? a.blist[blockIdx.x] : blockIdx.x;
      nb_e0 = a.boff[bi]; nb_e1 = a.boff[bi + 1]; nb_g0 = a.goff[bi]; nb_g1 = a.goff[bi + 1];
    }
    for (int b = blockIdx.x; b < nbl; b += G, ++it) {
      const int s = it & 1;
      const int e0 = nb_e0, Eb = nb_e1 - nb_e0, g0 = nb_g0, Gb = nb_g1 - nb_g0;
      if (b + G < nbl) {  // next block's metadata (consumed one iteration later)
        const int bi = a.blist ? a.blist[b + G] : b + G;
        nb_e0 = a.boff[bi]; nb_e1 = a.boff[bi + 1]; nb_g0 = a.goff[bi]; nb_g1 = a.goff[bi + 1];
      }
      // ghost ids (lane g holds ghost g and g + 32) and neighbour slots of own elements lane, lane + 32
      const int gl0 = (lane < Gb) ? a.gid[g0 + lane] : 0;
      const int gl1 = (lane + 32 < Gb) ? a.gid[g0 + lane + 32] : 0;
      const short4 zs = make_short4(0, 0, 0, 0);
      const short4 nb0 = (lane < Eb) ? a.nbr[e0 + lane] : zs;
      const short4 nb1 = (lane + 32 < Eb) ? a.nbr[e0 + lane + 32] : zs;
      if (it >= 2) mbar_wait(empty + s, ((it >> 1) + 1) & 1);
      double* sb = sm + L.stg + s * L.sz;
      const int64_t g0n = (int64_t)e0 * NP;
      const int shift = (int)(g0n & 1);
      double* rows = sb + L.o_rows + shift;   // slot s row at rows + s * NP
      double* prow = sm + L.pold + shift;
      double* gG = sb + L.o_gG;
      // ghost rows (8-byte copies: any alignment) and records; halo ghosts (id >= K) read the received
      // rows, their p_{k-1} is zero (the received rows are p_k already)
      for (int q0 = 0; q0 < Gb * NP; q0 += 32) {  // warp-uniform trip count (the shuffles need every lane)
        const int q = q0 + lane;
        const int g = q / NP, i = q - g * NP;
        const int v0 = __shfl_sync(0xffffffffu, gl0, g & 31), v1 = __shfl_sync(0xffffffffu, gl1, g & 31);
        if (q >= Gb * NP) continue;
        const int ge = (g < 32) ? v0 : (g < 64) ? v1 : a.gid[g0 + g];
        const bool halo = ge >= K;
        const int64_t off = (halo ? (int64_t)(ge - K) : (int64_t)ge) * NP + i;
        cp_async8(rows + (E + g) * NP + i, (halo ? a.halo_p : U) + off);
        if (with_p) cp_async8(prow + (E + g) * NP + i, halo ? a.zero_row + i : pold + off);
      }
      for (int g = lane; g < Gb; g += 32) {
        const int ge = (g < 32) ? gl0 : (g < 64) ? gl1 : a.gid[g0 + g];
        cp_async16(gG + (E + g) * 4, reinterpret_cast<const double*>(a.gG + ge));
        cp_async16(gG + (E + g) * 4 + 2, reinterpret_cast<const double*>(a.gG + ge) + 2);
      }
      // own rows: one contiguous range per vector by TMA bulk copy (16-byte aligned: the copy starts one
      // double early when the range starts on an odd double); the array's tail block falls back to cp.async
      const int64_t gbase = g0n - shift;
      const unsigned nbytes = (unsigned)(((Eb * NP + shift) * 8 + 15) & ~15);
      const bool tma = (gbase + nbytes / 8 <= K * NP);
      if (!tma) {
        for (int q = lane; q < Eb * NP; q += 32) {
          cp_async8(rows + q, U + g0n + q);
          if (with_p) cp_async8(prow + q, pold + g0n + q);
        }
      }
      // face descriptors of the own elements: x = trace-row base of the other side (its slot row and
      // face column block; the element itself, mirrored, on a physical boundary), y = flip | bc << 1
      int2* fd = reinterpret_cast<int2*>(sb + L.o_fd);
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int e = lane + 32 * r;
        if (e < Eb) {
          const short4 nb = r ? nb1 : nb0;
#pragma unroll
          for (int f = 0; f < 3; ++f) {
            const int fl = (nb.w >> (4 * f)) & 15;
            const int fp = fl & 3, bc = fl >> 2;
            const int slot = (f == 0) ? nb.x : (f == 1) ? nb.y : nb.z;
            const bool inner = (bc == 0);
            const int flip = inner && ((f == 2) == (fp == 2));
            fd[3 * e + f] = make_int2(inner ? slot * TS + fp * NFP : e * TS + f * NFP, flip | (bc << 1));
          }
        }
      }
      if (lane == 0) {
        int* meta = reinterpret_cast<int*>(sb + L.o_meta);
        meta[0] = e0;
        meta[1] = Eb;
        meta[2] = Gb;
      }
      __syncwarp();  // the warp's shared-memory stores before lane 0's release arrival
      if (lane == 0) {
        const unsigned rec = (unsigned)Eb * 32u + (unsigned)Eb * (8u * GF);
        mbar_expect_tx(full + s, rec + (tma ? nbytes * (1u + (with_p ? 1u : 0u)) : 0u));
        tma_load_1d(gG, a.gG + e0, (unsigned)Eb * 32u, full + s);
        tma_load_1d(sb + L.o_gF, a.gF + (int64_t)e0 * GF, (unsigned)Eb * (8u * GF), full + s);
        if (tma) {
          tma_load_1d(sb + L.o_rows, U + gbase, nbytes, full + s);
          if (with_p) tma_load_1d(sm + L.pold, pold + gbase, nbytes, full + s);
        }
      }
      cp_async_mbar_arrive_noinc(full + s);  // arrives once this lane's cp.async copies have landed
      if (PCG) {
        // p_k = z + beta p_{k-1} in place (own and ghost rows), p_k and x += alpha_{k-1} p_{k-1} of the own
        // rows to global (coalesced); then the compute warps may start (ready)
        mbar_wait(full + s, (it >> 1) & 1);
        const int no = Eb * NP;
        constexpr int B8 = 8;
        for (int q0 = 0; q0 < no; q0 += 32 * B8) {
          double xv[B8];
#pragma unroll
          for (int u = 0; u < B8; ++u) {
            const int q = q0 + 32 * u + lane;
            xv[u] = (with_x && q < no) ? a.x[g0n + q] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < B8; ++u) {
            const int q = q0 + 32 * u + lane;
            if (q < no) {
              const double po = prow[q];
              const double v = fma(beta, po, rows[q]);
              rows[q] = v;
              pnew[g0n + q] = v;
              if (with_x) a.x[g0n + q] = fma(alpha_prev, po, xv[u]);
            }
          }
        }
        for (int q = lane; q < Gb * NP; q += 32) rows[E * NP + q] = fma(beta, prow[E * NP + q], rows[E * NP + q]);
        __syncwarp();
        if (lane == 0) mbar_arrive(ready + s);
      }
    }
  } else {
    // ================================================================ compute warps
    // per-lane tables: trace columns of the C-fragment nodes 8 nt + 2 (lane & 3) + h and of the A-fragment
    // nodes 4 kc + (lane & 3) (for u); face-node items of P2 (4 lanes per element): fk = 4q + (lane & 3)
    int tcol[2 * NT];
#pragma unroll
    for (int q = 0; q < 2 * NT; ++q) tcol[q] = node_trace_cols<N>(8 * (q >> 1) + 2 * (lane & 3) + (q & 1), T::NF3 + (lane & 3));
    int ucol[KCG];
#pragma unroll
    for (int kc = 0; kc < KCG; ++kc) ucol[kc] = node_trace_cols<N>(4 * kc + (lane & 3), T::NF3 + (lane & 3));
    int itab[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int fk = 4 * q + (lane & 3);
      const int f = fk / NFP, kk = fk - f * NFP;
      itab[q] = (fk < T::NF3) ? ((f << 8) | kk) : ((2 << 8) | N);
    }
    int it = 0;
    for (int b = blockIdx.x; b < nbl; b += G, ++it) {
      const int s = it & 1;
      const double* sb = sm + L.stg + s * L.sz;
      mbar_wait(PCG ? ready + s : full + s, (it >> 1) & 1);
      const int* meta = reinterpret_cast<const int*>(sb + L.o_meta);
      const int64_t e0 = meta[0];
      const int Eb = meta[1], Gb = meta[2];
      const double* rows = sb + L.o_rows + (int)((e0 * NP) & 1);
      const double* gGs = sb + L.o_gG;
      const double* gFs = sb + L.o_gF;
      const int2* fds = reinterpret_cast<const int2*>(sb + L.o_fd);
      if (it > 0) named_bar_sync(1, NCT);  // every compute warp is done reading the traces of block b - G

      // ---- P1: reference gradient of a tile of 8 slot rows on DMMA; face traces -sJ n.grad u and u
      // at the face nodes to the trace rows
      auto store_traces = [&](int srow, const double (&acc)[2 * NT][2], double (*wr)[2], double (*ws)[2]) {
        const double* gq = gGs + srow * 4;
        const double Grr = gq[0], Grs = gq[1], Gss = gq[2];
        double* trow = trc + srow * TS;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double ur = acc[nt][h], us = acc[NT + nt][h];
            const double wrv = Grr * ur + Grs * us, wsv = Grs * ur + Gss * us;
            const int c = tcol[2 * nt + h];
            trow[c & 31] = wsv;
            trow[(c >> 5) & 31] = -(wrv + wsv);
            trow[(c >> 10) & 31] = wrv;
            if (wr) {
              wr[nt][h] = wrv;
              ws[nt][h] = wsv;
            }
          }
      };
      auto load_a = [&](int srow, double (&av)[KCG]) {
        double* trow = trc + srow * TS + UO;
#pragma unroll
        for (int kc = 0; kc < KCG; ++kc) {
          const int i = 4 * kc + (lane & 3);
          av[kc] = (i < NP) ? rows[srow * NP + i] : 0.0;
          const int c = ucol[kc];
          trow[c & 31] = av[kc];
          trow[(c >> 5) & 31] = av[kc];
          trow[(c >> 10) & 31] = av[kc];
        }
      };
      const int t0 = TT * warp;
      const int nown = min(TT, max(0, (Eb - 8 * t0 + 7) / 8));  // active own tiles of this warp
      double wr[TT][NT][2], ws[TT][NT][2];
      {
        double av[TT][KCG];
#pragma unroll
        for (int t = 0; t < TT; ++t)
          if (t < nown) load_a(8 * (t0 + t) + (lane >> 2), av[t]);
        double acc[TT][2 * NT][2];
#pragma unroll
        for (int t = 0; t < TT; ++t)
#pragma unroll
          for (int q = 0; q < 2 * NT; ++q) acc[t][q][0] = acc[t][q][1] = 0.0;
        if (nown == TT) {
#pragma unroll
          for (int kc = 0; kc < KCG; ++kc) {
            const double* bt = tabG + kc * 2 * NT * 32 + lane;
#pragma unroll
            for (int q = 0; q < 2 * NT; ++q) {
              const double bv = bt[q * 32];
#pragma unroll
              for (int t = 0; t < TT; ++t) dmma(acc[t][q][0], acc[t][q][1], av[t][kc], bv);
            }
          }
        } else if (nown > 0) {
#pragma unroll
          for (int kc = 0; kc < KCG; ++kc) {
            const double* bt = tabG + kc * 2 * NT * 32 + lane;
#pragma unroll
            for (int q = 0; q < 2 * NT; ++q) dmma(acc[0][q][0], acc[0][q][1], av[0][kc], bt[q * 32]);
          }
        }
#pragma unroll
        for (int t = 0; t < TT; ++t)
          if (t < nown) store_traces(8 * (t0 + t) + (lane >> 2), acc[t], wr[t], ws[t]);
      }
      // ---- P1 ghost tiles, round robin over the compute warps (traces only)
      const int ngt = (Gb + 7) / 8;
      for (int gt = warp; gt < ngt; gt += WC) {
        const int srow = E + 8 * gt + (lane >> 2);
        double av[KCG];
        load_a(srow, av);
        double acc[2 * NT][2];
#pragma unroll
        for (int q = 0; q < 2 * NT; ++q) acc[q][0] = acc[q][1] = 0.0;
#pragma unroll
        for (int kc = 0; kc < KCG; ++kc) {
          const double* bt = tabG + kc * 2 * NT * 32 + lane;
#pragma unroll
          for (int q = 0; q < 2 * NT; ++q) dmma(acc[q][0], acc[q][1], av[kc], bt[q * 32]);
        }
        store_traces(srow, acc, nullptr, nullptr);
      }
      // ---- P3 volume part of the own tiles, from registers (before the barrier)
      double C[TT][NT][2];
#pragma unroll
      for (int t = 0; t < TT; ++t)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) C[t][nt][0] = C[t][nt][1] = 0.0;
      if (nown > 0) {
#pragma unroll
        for (int c = 0; c < 2 * NT; ++c) {
          const double* bt = tabM + c * NT * 32 + lane;
          const double* bu = tabM + (2 * NT + c) * NT * 32 + lane;
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const double b1 = bt[j * 32];
#pragma unroll
            for (int t = 0; t < TT; ++t)
              if (t < nown) dmma(C[t][j][0], C[t][j][1], wr[t][c >> 1][c & 1], b1);
          }
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const double b2 = bu[j * 32];
#pragma unroll
            for (int t = 0; t < TT; ++t)
              if (t < nown) dmma(C[t][j][0], C[t][j][1], ws[t][c >> 1][c & 1], b2);
          }
        }
      }
      named_bar_sync(1, NCT);  // the traces of every slot are written

      // ---- P2 + P3 face part of the own tiles (TT per warp, shared B fragments)
      if (nown > 0) {
        int ec[TT];
#pragma unroll
        for (int t = 0; t < TT; ++t) {
          const int e = 8 * (t0 + t) + (lane >> 2);
          ec[t] = e < Eb ? e : 8 * t0;  // rows past the block end compute on a valid slot, never stored
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int f = itab[q] >> 8, kk = itab[q] & 255;
          double far[TT], fas[TT], fag[TT];
#pragma unroll
          for (int t = 0; t < TT; ++t) {
            const int2 dsc = fds[3 * ec[t] + f];
            const int flip = dsc.y & 1, bc = dsc.y >> 1;
            const int kq = flip ? NFP - 1 - kk : kk;
            const double* to = trc + ec[t] * TS + f * NFP + kk;
            const double tm = to[0];                     // -sJ n-.grad u-
            const double um = to[UO];                    // u-
            const double tp = trc[dsc.x + kq];           // -sJ n+.grad u+ (the other side's own normal)
            const double up = trc[dsc.x + UO + kq];      // u+ (before mirroring)
            const double* fq = gFs + ec[t] * GF + 3 * f;
            // boundary faces read the element's own traces and mirror them (R7):
            // Dirichlet u+ = -u-, grad u+ = grad u-;  Neumann u+ = u-, grad u+ = -grad u-
            const double delta = ((bc == 1) ? -up : up) - um;   // paper jump
            far[t] = fq[0] * delta;                              // 1/2 sJ (n.grad r) delta
            fas[t] = fq[1] * delta;                              // 1/2 sJ (n.grad s) delta
            const double hp = (bc == 1) ? 0.5 : -0.5;
            fag[t] = fma(0.5, tm, fma(hp, tp, -fq[2] * delta));  // -sJ (n-.{grad u} + tau delta)
          }
          const double* b0 = tabM + (KCW + q) * NT * 32 + lane;
          const double* b1 = tabM + (KCW + NQ + q) * NT * 32 + lane;
          const double* b2 = tabM + (KCW + 2 * NQ + q) * NT * 32 + lane;
          // chains interleaved: consecutive DMMAs go to different accumulators (26.6-cycle DMMA latency)
#pragma unroll
          for (int m = 0; m < 3; ++m) {
            const double* bm = (m == 0) ? b0 : (m == 1) ? b1 : b2;
#pragma unroll
            for (int j = 0; j < NT; ++j) {
              const double v = bm[j * 32];
#pragma unroll
              for (int t = 0; t < TT; ++t)
                if (t < nown) dmma(C[t][j][0], C[t][j][1], (m == 0) ? far[t] : (m == 1) ? fas[t] : fag[t], v);
            }
          }
        }
        if (LAM) {
#pragma unroll
          for (int kc = 0; kc < KCM; ++kc) {
            const int i = 4 * kc + (lane & 3);
            const double* bt = tabL + kc * NT * 32 + lane;
            double av[TT];
#pragma unroll
            for (int t = 0; t < TT; ++t) av[t] = (i < NP) ? a.lambda * gGs[ec[t] * 4 + 3] * rows[ec[t] * NP + i] : 0.0;
#pragma unroll
            for (int j = 0; j < NT; ++j) {
              const double bv = bt[j * 32];
#pragma unroll
              for (int t = 0; t < TT; ++t)
                if (t < nown) dmma(C[t][j][0], C[t][j][1], av[t], bv);
            }
          }
        }
#pragma unroll
        for (int t = 0; t < TT; ++t) {
          const int e = 8 * (t0 + t) + (lane >> 2);
          if (t < nown && e < Eb) {
            const int64_t base = (e0 + e) * NP;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int i = 8 * nt + 2 * (lane & 3) + h;
                if (i < NP) {
                  a.Au[base + i] = C[t][nt][h];
                  if (PCG) dot += rows[e * NP + i] * C[t][nt][h];
                }
              }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);  // this warp is done with stage s
    }
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
}

}  // namespace ipdg
