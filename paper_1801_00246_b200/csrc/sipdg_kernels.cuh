// FP64 SIPDG operator, Jacobi diagonal and PCG vector kernels for sm_100a.
// Paper: arXiv:1801.00246 (P:n = PAPER.md line n).  Formulation in kernels.cuh.
//
// Kernel k_sipdg<N, MODE, LAM> (persistent CTAs, W warps, loop over element blocks):
//   per element block of <= E = 8W own elements plus the block's G ghost elements
//   (face neighbours outside the block, listed at setup):
//   P0  u of own + ghost elements -> smem (Ax: cp.async; PCG pass A: p = D^-1 r + beta p_{k-1}
//       formed from batched loads, p_k and the deferred x update written back);
//       per-slot face geometry (J, det G, unit normals, sJ) computed once per slot
//   P1  per 8-element tile: [u_r | u_s] = u [Dr^T | Ds^T] on DMMA      (Alg. AxG);
//       w_r, w_s = J G (u_r, u_s) -> smem (they also give the face normal derivatives) and, for
//       own tiles, stay in registers (C layout) as the A operand of P3
//   P2  per own face node: delta = u+ - u- (mirrored on boundary faces), flux
//       g = 1/2 n-.(grad u- + grad u+) + tau delta                     (Alg. AxKernel)
//       -> face block [1/2 sJ (n.grad r) delta | 1/2 sJ (n.grad s) delta | -sJ g]
//   P3  per own tile: Au = [w_r | w_s | face block] x [Sr; Ss; LIFT^T Sr; LIFT^T Ss; E^T] on DMMA
//       (+ lambda J u M), stored element-major; PCG pass A also accumulates p . Ap.
#pragma once
#include "kernels.cuh"

namespace ipdg {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_group1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on an mbarrier
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n"
      ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

enum { MODE_AX = 0, MODE_PCG_A = 1 };

// Optional phase timing (compile with -DIPDG_PHASE_TIMING; tools/phase_timing.py): warp 0 of every
// CTA accumulates clock64() deltas per phase into ipdg_phase_cycles[8].
#ifdef IPDG_PHASE_TIMING
static __device__ unsigned long long ipdg_phase_cycles[8];
#define PHASE_MARK(id)                                                   \
  do {                                                                   \
    if (threadIdx.x == 0) {                                              \
      const long long t_ = clock64();                                    \
      atomicAdd(&ipdg_phase_cycles[id], (unsigned long long)(t_ - ph_t)); \
      ph_t = t_;                                                         \
    }                                                                    \
  } while (0)
#else
#define PHASE_MARK(id) do { } while (0)
#endif

// shared-memory layout (in doubles) shared by host and device
struct SmemLayout {
  int tabG, tabM, tabL, iaux, us, geo, fg, nb, gid, wsm, stg, mbar, total;  // offsets in doubles
  template <int N>
  __host__ __device__ static SmemLayout make(int gmax, bool lam, bool pcg) {
    using T = Tr<N>;
    SmemLayout L;
    const int gm8 = (gmax + 7) / 8 * 8;
    const int slots = T::E + gm8;
    int o = 0;
    L.tabG = o; o += T::TAB_G;
    L.tabM = o; o += T::TAB_M;
    L.tabL = o; o += lam ? T::TAB_L : 0;
    L.iaux = o; o += (6 * T::NFP + 1) / 2;  // ints: neighbour face-node index nidx[f'][flip][k]
    o = (o + 1) & ~1;                   // 16-byte alignment
    L.us = o; o += slots * T::SU;
    o = (o + 1) & ~1;
    L.geo = o; o += slots * T::SG;
    L.fg = o; o += 9 * T::FGS;         // own elements: per face c_r c_s sJ*tau, layout [3f + field][e]
    L.nb = o; o += 2 * T::E;            // short4 per element, double-buffered
    L.gid = o; o += gm8;                // 2 x gm8 ints, double-buffered
    o = (o + 1) & ~1;
    L.wsm = o; o += slots * T::SXY;     // w_r | w_s per slot (the face block lives in registers)
    // PCG staging of z, p_{k-1}, x (own) and z, p_{k-1} (ghosts) aliases wsm, which is produced
    // only after the staging has been consumed
    L.stg = L.wsm;
    const int need = pcg ? 3 * (T::E * T::NP + 2) + 2 * gm8 * T::NP : 0;  // own arrays padded for TMA alignment
    if (L.stg + need > o) o = L.stg + need;
    L.mbar = o; o += 1;
    L.total = o;
    return L;
  }
};

// copy loop over element rows: warp-strided rows, lanes across the Np entries of a row
template <int N, class F>
__device__ __forceinline__ void for_rows(int nrows, int warp, int lane, F&& f) {
  using T = Tr<N>;
  constexpr int NP = T::NP, RPW = T::RPW, W = T::W;
  const int rsub = (NP >= 32) ? 0 : lane / NP;
  const int i0 = (NP >= 32) ? lane : lane - rsub * NP;
  if (rsub >= RPW) return;
  for (int row = warp * RPW + rsub; row < nrows; row += W * RPW) {
#pragma unroll
    for (int ps = 0; ps < T::NPASS; ++ps) {
      const int i = i0 + 32 * ps;
      if (i < NP) f(row, i);
    }
  }
}

// deterministic block reduction of NV doubles; result valid in thread 0
template <int NV>
__device__ __forceinline__ void block_reduce(double (&v)[NV], double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) red[warp * NV + q] = v[q];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += red[w * NV + q];
      v[q] = s;
    }
  }
}

// grid-level deterministic reduction: partials[blockIdx] then the last CTA sums in index order.
// Returns true in thread 0 of the last CTA, with `out` holding the totals.
template <int NV>
__device__ bool grid_reduce(double (&v)[NV], double* red, double* partials, unsigned int* counter, double (&out)[NV]) {
  block_reduce<NV>(v, red);
  __shared__ bool am_last;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) partials[q * gridDim.x + blockIdx.x] = v[q];
    __threadfence();
    const unsigned int t = atomicAdd(counter, 1u);
    am_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  double w[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double s = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) s += ((volatile double*)partials)[q * gridDim.x + i];
    w[q] = s;
  }
  block_reduce<NV>(w, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) out[q] = w[q];
    *counter = 0u;
  }
  return threadIdx.x == 0;
}

template <int N, int MODE, bool LAM>
__global__ void __launch_bounds__(Tr<N>::W * 32, Tr<N>::MINB) k_sipdg(AxArgs a, int gmax) {
  using T = Tr<N>;
  constexpr int NP = T::NP, NFP = T::NFP, NF3 = T::NF3, NT = T::NT, NPN = T::NPN, SU = T::SU, SF = T::SF;
  constexpr int SXY = T::SXY, SG = T::SG;
  constexpr int W = T::W, E = T::E, KCG = T::KCG, KCW = T::KCW, KCF = T::KCF, KCM = T::KCM;
  constexpr int NTHR = W * 32;
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[32 * 3];
  const SmemLayout L = SmemLayout::make<N>(gmax, LAM, MODE == MODE_PCG_A);
  const int gm8 = (gmax + 7) / 8 * 8;
  double* tabG = sm + L.tabG;
  double* tabM = sm + L.tabM;
  double* tabL = sm + L.tabL;
  int* nidx = reinterpret_cast<int*>(sm + L.iaux);
  double* us = sm + L.us;
  double* geos = sm + L.geo;
  double* fgs = sm + L.fg;
  short4* nbs0 = reinterpret_cast<short4*>(sm + L.nb);
  int* gids0 = reinterpret_cast<int*>(sm + L.gid);
  double* wsm = sm + L.wsm;
  double* stg = sm + L.stg;
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(sm + L.mbar);
  unsigned mbar_phase = 0;
  constexpr int OSTR = E * NP + 2;  // own staging array stride (TMA head alignment pad)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t K = a.K;

  // ---- PCG pass-A prologue: decisions from the previous iteration's reductions
  double beta = 0.0, alpha_prev = 0.0, dot = 0.0;
  bool first = false, stop = false, zero_x = false, do_xupd = false;
  long long k = 0;
  int new_status = 0;
  double rhoB = 0.0, rrB = 0.0, bbv = 0.0;
  double* pnew = nullptr;
  const double* pold = nullptr;
  if (MODE == MODE_PCG_A) {
    PcgState* st = a.st;
    if (st->stop_iter >= 0) return;  // stopped by an earlier launch
    k = st->it + 1;
    first = (k == 1);
    pnew = (k & 1) ? a.p_odd : a.p_even;
    pold = (k & 1) ? a.p_even : a.p_odd;
    rhoB = st->red_B[0];
    rrB = st->red_B[1];
    bbv = first ? st->red_B[2] : st->bb;
    if (first) {
      if (bbv == 0.0) { stop = true; zero_x = true; }
      else if (rrB <= st->tol2 * bbv) stop = true;
      else if (st->maxit == 0) { stop = true; new_status = 1; }
    } else {
      if (rrB <= st->tol2 * bbv) stop = true;
      else if (k - 1 >= st->maxit) { stop = true; new_status = 1; }
      alpha_prev = st->rho_hist[(k - 2) & 3] / st->red_A;
      do_xupd = true;
      beta = rhoB / st->rho_hist[(k - 2) & 3];
    }
    if (stop) {
      const int64_t n = K * NP;
      for (int64_t i = blockIdx.x * (int64_t)NTHR + tid; i < n; i += (int64_t)gridDim.x * NTHR) {
        if (zero_x) a.x[i] = 0.0;
        else if (do_xupd) a.x[i] += alpha_prev * pold[i];
      }
      double v[1] = {0.0}, out[1];
      if (grid_reduce<1>(v, red, a.partials, a.counter, out)) {
        st->stop_iter = k - 1;
        st->status = new_status;
        st->final_rr = rrB;
        if (first) st->bb = bbv;
      }
      return;
    }
  }

  // ---- once per CTA: operator tables, index table, zero padding; neighbour data of block 0
  {
    const double* src = a.tables;
    constexpr int ntab = T::TAB_G + T::TAB_M + (LAM ? T::TAB_L : 0);  // multiple of 32 doubles
    for (int i = 2 * tid; i < ntab; i += 2 * NTHR) cp_async16(sm + i, src + i);
    for (int q = tid; q < 6 * NFP; q += NTHR) {  // nidx[fp][flip][k] = Fmask[fp][flip ? Nfp-1-k : k]
      const int fp = q / (2 * NFP), fl = (q / NFP) & 1, kk = q % NFP;
      nidx[q] = fmask_cf<N>(fp, fl ? NFP - 1 - kk : kk);
    }
    const int slots = E + gm8;
    for (int i = tid; i < slots * SU; i += NTHR) us[i] = 0.0;
    if (MODE == MODE_PCG_A && tid == 0) {
      mbar_init(mbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    const int b = blockIdx.x;
    if (b < a.nblocks) {
      const int e0 = a.boff[b], Eb = a.boff[b + 1] - e0, g0 = a.goff[b], Gb = a.goff[b + 1] - g0;
      for (int e = tid; e < Eb; e += NTHR) cp_async8(nbs0 + e, a.nbr + e0 + e);
      for (int g = tid; g < Gb; g += NTHR) gids0[g] = a.gid[g0 + g];
    }
  }

  // face-node items of this lane (4 lanes per element): fk = 4q + (lane & 3) -> (f, k, node)
  int itab[T::NQ];
#pragma unroll
  for (int q = 0; q < T::NQ; ++q) {
    const int fk = 4 * q + (lane & 3);
    const int f = fk / NFP, kk = fk - f * NFP;
    itab[q] = (fk < NF3) ? ((f << 24) | (kk << 16) | fmask_cf<N>(f, kk)) : -1;
  }
  double wr[NT][2], ws[NT][2];
  int par = 0;
#ifdef IPDG_PHASE_TIMING
  long long ph_t = clock64();
#endif
  int cur_e0 = 0, cur_Eb = 0, cur_Gb = 0;  // block metadata, prefetched one block ahead
  if (blockIdx.x < a.nblocks) {
    cur_e0 = a.boff[blockIdx.x];
    cur_Eb = a.boff[blockIdx.x + 1] - cur_e0;
    cur_Gb = a.goff[blockIdx.x + 1] - a.goff[blockIdx.x];
  }
  for (int b = blockIdx.x; b < a.nblocks; b += gridDim.x, par ^= 1) {
    const int64_t e0 = cur_e0;
    const int Eb = cur_Eb;
    const int Gb = cur_Gb;
    short4* nbs = nbs0 + par * E;
    int* gids = gids0 + par * gm8;
    int own_shift = 0;
    bool use_tma = false;
    cp_async_wait_all();
    __syncthreads();  // previous block done with the buffers; this block's gids / nbr landed
    PHASE_MARK(0);  // wait for the previous block's stragglers + this block's metadata
    // ---- P0: async copies of the element data of this block
    for (int q = tid; q < 2 * (Eb + Gb); q += NTHR) {  // raw geometry r_x s_x r_y s_y (2 x 16 B)
      const int s = q >> 1, h = q & 1;
      const int slot = s < Eb ? s : E + (s - Eb);
      const int64_t el = s < Eb ? e0 + s : (int64_t)gids[s - Eb];
      cp_async16(geos + slot * SG + 2 * h, reinterpret_cast<const double*>(a.geo + el) + 2 * h);
    }
    if (MODE == MODE_AX) {
      const double* u = a.u;
      for_rows<N>(Eb, warp, lane, [&](int e, int i) { cp_async8(us + e * SU + i, u + (e0 + e) * NP + i); });
      for_rows<N>(Gb, warp, lane, [&](int g, int i) {
        const int ge = gids[g];
        const double* srcp = ge >= K ? a.halo_p + (int64_t)(ge - K) * NP : u + (int64_t)ge * NP;
        cp_async8(us + (E + g) * SU + i, srcp + i);
      });
    } else {
      // own rows: one contiguous range per vector -> TMA bulk copies (16-byte aligned: the copy
      // starts one double early when the range starts on an odd double; the tail block of the
      // arrays falls back to cp.async)
      double* sz = stg;                  // own: z | p_{k-1} | x (stride OSTR), then ghosts: z | p_{k-1}
      double* sp = stg + OSTR;
      double* sx = stg + 2 * OSTR;
      double* gz = stg + 3 * OSTR;
      double* gp = gz + gm8 * NP;
      const int64_t g0 = e0 * NP;
      own_shift = (int)(g0 & 1);
      const int64_t gb = g0 - own_shift;
      const unsigned nbytes = (unsigned)(((Eb * NP + own_shift) * 8 + 15) & ~15);
      use_tma = (gb + nbytes / 8 <= K * NP);
      if (use_tma) {
        if (tid == 0) {
          const unsigned tot = nbytes * (1u + (first ? 0u : 1u) + (do_xupd ? 1u : 0u));
          mbar_expect_tx(mbar, tot);
          tma_load_1d(sz, a.z + gb, nbytes, mbar);
          if (!first) tma_load_1d(sp, pold + gb, nbytes, mbar);
          if (do_xupd) tma_load_1d(sx, a.x + gb, nbytes, mbar);
        }
      } else {
        own_shift = 0;
        for_rows<N>(Eb, warp, lane, [&](int e, int i) {
          const int64_t g = (e0 + e) * NP + i;
          cp_async8(sz + e * NP + i, a.z + g);
          if (!first) cp_async8(sp + e * NP + i, pold + g);
          if (do_xupd) cp_async8(sx + e * NP + i, a.x + g);
        });
      }
      for_rows<N>(Gb, warp, lane, [&](int q, int i) {
        const int ge = gids[q];
        if (ge >= K) {
          cp_async8(gz + q * NP + i, a.halo_p + (int64_t)(ge - K) * NP + i);
        } else {
          const int64_t g = (int64_t)ge * NP + i;
          cp_async8(gz + q * NP + i, a.z + g);
          if (!first) cp_async8(gp + q * NP + i, pold + g);  // p_{k-1}; owners write p_k elsewhere
        }
      });
    }
    cp_async_commit();
    // prefetch the neighbour slots / ghost ids of this CTA's next block (small, double-buffered)
    {
      const int bn = b + gridDim.x;
      if (bn < a.nblocks) {
        const int e0n = a.boff[bn], Ebn = a.boff[bn + 1] - e0n, g0n = a.goff[bn], Gbn = a.goff[bn + 1] - g0n;
        short4* nbn = nbs0 + (par ^ 1) * E;
        int* gin = gids0 + (par ^ 1) * gm8;
        for (int e = tid; e < Ebn; e += NTHR) cp_async8(nbn + e, a.nbr + e0n + e);
        for (int g = tid; g < Gbn; g += NTHR) cp_async4(gin + g, a.gid + g0n + g);
        cur_e0 = e0n;
        cur_Eb = Ebn;
        cur_Gb = Gbn;
      }
      cp_async_commit();
    }
    cp_async_wait_group1();  // this block's data complete; the prefetch may still fly
    if (MODE == MODE_PCG_A && use_tma) {
      mbar_wait(mbar, mbar_phase);
      mbar_phase ^= 1u;
    }
    __syncthreads();
    if (MODE == MODE_PCG_A) {  // p_k = z + beta p_{k-1} (own + ghosts); x += alpha_{k-1} p_{k-1}
      const double* sz = stg + own_shift;
      const double* sp = stg + OSTR + own_shift;
      const double* sx = stg + 2 * OSTR + own_shift;
      const double* gz = stg + 3 * OSTR;
      const double* gp = gz + gm8 * NP;
      for_rows<N>(Eb, warp, lane, [&](int e, int i) {
        const int o = e * NP + i;
        const double po = first ? 0.0 : sp[o];
        const double v = sz[o] + beta * po;
        const int64_t g = (e0 + e) * NP + i;
        pnew[g] = v;
        if (do_xupd) a.x[g] = sx[o] + alpha_prev * po;
        us[e * SU + i] = v;
      });
      for_rows<N>(Gb, warp, lane, [&](int q, int i) {
        const int o = q * NP + i;
        const double v = (gids[q] >= K || first) ? gz[o] : gz[o] + beta * gp[o];
        us[(E + q) * SU + i] = v;
      });
      __syncthreads();
    }

    PHASE_MARK(1);  // P0: loads (and PCG prep)
    // ---- P1: reference gradient on DMMA; w_r / w_s to smem, and kept in registers for own tiles
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
      double* gq = geos + srow * SG;
      const double rx = gq[0], sx = gq[1], ry = gq[2], sy = gq[3];
      const double det = rx * sy - sx * ry;  // = 1/J
      const double J = 1.0 / det;
      if ((lane & 3) == 0) { gq[4] = J; gq[5] = det; }
      if (own && (lane & 3) < 3 && srow < Eb) {  // one face per lane: lift coefficients and sJ * tau
        const int f = lane & 3;
        const double gx = (f == 0) ? -sx : (f == 1) ? rx + sx : -rx;  // outward: -grad s, grad r+s, -grad r
        const double gy = (f == 0) ? -sy : (f == 1) ? ry + sy : -ry;
        const double sJ = J * sqrt(gx * gx + gy * gy);                 // edge length / 2 (R6)
        const short4 nb = nbs[srow];
        const int bc = (nb.w >> (4 * f + 2)) & 3;
        double detp = 0.0;                                             // neighbour det G (= 1/J+) on interior faces
        if (bc == 0) {
          const double* gn = geos + ((f == 0) ? nb.x : (f == 1) ? nb.y : nb.z) * SG;
          detp = gn[0] * gn[3] - gn[1] * gn[2];
        }
        double* fq = fgs + 3 * f * T::FGS + srow;
        fq[0] = 0.5 * J * (rx * gx + ry * gy);                          // 1/2 sJ (n . grad r)
        fq[T::FGS] = 0.5 * J * (sx * gx + sy * gy);                     // 1/2 sJ (n . grad s)
        fq[2 * T::FGS] = sJ * a.tau_c * sJ * fmax(det, detp);           // sJ tau, Eq. Ch2.PenaltyParameter (1/h = sJ/J)
      }
      // w_r = J (G_rr u_r + G_rs u_s), w_s = J (G_rs u_r + G_ss u_s).  They are also the scaled
      // normal derivatives at the face nodes: J g_f . grad u with g_f = -grad s, grad r + grad s,
      // -grad r gives sJ (n . grad u) = -w_s, w_r + w_s, -w_r on faces 0, 1, 2.
      const double Grr = J * (rx * rx + ry * ry), Grs = J * (rx * sx + ry * sy), Gss = J * (sx * sx + sy * sy);
      double* wrow = wsm + srow * SXY + 2 * (lane & 3);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double ur0 = acc[nt][0], ur1 = acc[nt][1], us0 = acc[NT + nt][0], us1 = acc[NT + nt][1];
        const double r0 = Grr * ur0 + Grs * us0, r1 = Grr * ur1 + Grs * us1;
        const double s0 = Grs * ur0 + Gss * us0, s1 = Grs * ur1 + Gss * us1;
        *reinterpret_cast<double2*>(wrow + 8 * nt) = make_double2(r0, r1);
        *reinterpret_cast<double2*>(wrow + NPN + 8 * nt) = make_double2(s0, s1);
        if (own) {
          wr[nt][0] = r0;
          wr[nt][1] = r1;
          ws[nt][0] = s0;
          ws[nt][1] = s1;
        }
      }
    }
    __syncthreads();

    PHASE_MARK(2);  // P1 incl. the barrier
    // ---- P2 + P3 per warp on its own tile (no block barrier in between)
    if (8 * warp < Eb) {
      // P3 starts with the volume part, Au = [w_r | w_s] x [Sr; Ss], straight from registers;
      // P2 then produces the face block one face-node pass at a time (four lanes per element, the
      // values land exactly where the A fragments need them: A[e = lane>>2][k = lane&3]) and each
      // pass is fed to the tensor cores at once, so the scalar face work overlaps the DMMAs.
      const int e = 8 * warp + (lane >> 2);
      double C[NT][2];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) C[nt][0] = C[nt][1] = 0.0;
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
      {
        const int ec = e < Eb ? e : 8 * warp;  // rows past the block end compute on a valid slot, never stored
        const short4 nb = nbs[ec];
        const double* uo = us + ec * SU;
        const double* wo = wsm + ec * SXY;
        const double* fq0 = fgs + ec;
#pragma unroll
        for (int q = 0; q < T::NQ; ++q) {
          double far = 0.0, fas = 0.0, fag = 0.0;
          const int it = itab[q];
          if (it >= 0) {
            const int f = it >> 24, kk = (it >> 16) & 255, i = it & 65535;
            const int fl = (nb.w >> (4 * f)) & 15;
            const int fp = fl & 3, bc = fl >> 2;
            const int slot = (f == 0) ? nb.x : (f == 1) ? nb.y : nb.z;
            const double* fq = fq0 + 3 * f * T::FGS;
            // boundary faces read the element's own trace and mirror it (R7):
            // Dirichlet u+ = -u-, grad u+ = grad u-;  Neumann u+ = u-, grad u+ = -grad u-
            const bool inner = (bc == 0);
            const int ps = inner ? slot : ec;
            const int pf = inner ? fp : f;
            const int ip = inner ? nidx[(2 * fp + ((f == 2) == (fp == 2))) * NFP + kk] : i;
            const double* wn = wsm + ps * SXY;
            const double um = uo[i], upr = us[ps * SU + ip];
            // sJ n.grad u at the node: -w_s, w_r + w_s, -w_r on faces 0, 1, 2 (own normal for u-,
            // the neighbour's own normal for u+, hence the sign flip below)
            const double wro = wo[i], wso = wo[NPN + i], wrn = wn[ip], wsn = wn[NPN + ip];
            const double tm = (f == 0) ? -wso : (f == 1) ? wro + wso : -wro;
            const double tp = (pf == 0) ? -wsn : (pf == 1) ? wrn + wsn : -wrn;
            const double tq = (bc == 1) ? tp : -tp;                 // sJ n-.grad u+ after mirroring
            const double delta = ((bc == 1) ? -upr : upr) - um;     // paper jump
            far = fq[0] * delta;                                    // 1/2 sJ (n.grad r) delta
            fas = fq[T::FGS] * delta;                               // 1/2 sJ (n.grad s) delta
            fag = -0.5 * (tm + tq) - fq[2 * T::FGS] * delta;        // -sJ (n.{grad u} + tau delta)
          }
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
      PHASE_MARK(3);  // P2 + P3 GEMM (warp 0)
      if (LAM) {
        const double lj = a.lambda * geos[e * SG + 4];
        const double* urow = us + e * SU + (lane & 3);
#pragma unroll
        for (int kc = 0; kc < KCM; ++kc) {
          const double av = lj * urow[4 * kc];
          const double* bt = tabL + kc * NT * 32 + lane;
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma(C[j][0], C[j][1], av, bt[j * 32]);
        }
      }
      PHASE_MARK(4);  // P3 GEMM (warp 0)
      if (e < Eb) {
        const int64_t base = (e0 + e) * NP;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int i = 8 * nt + 2 * (lane & 3) + h;
            if (i < NP) {
              a.Au[base + i] = C[nt][h];
              if (MODE == MODE_PCG_A) dot += us[e * SU + i] * C[nt][h];
            }
          }
      }
      PHASE_MARK(5);  // P3 stores (warp 0)
    }
  }
  cp_async_wait_all();
  if (MODE == MODE_PCG_A) {
    double v[1] = {dot}, out[1];
    if (grid_reduce<1>(v, red, a.partials, a.counter, out)) {
      PcgState* st = a.st;
      st->red_A = out[0];
      st->rho_hist[(k - 1) & 3] = rhoB;
      if (first) st->bb = bbv;
    }
  }
}

// ---- PCG pass B: r -= alpha A p; z = D^{-1} r; partial (r.z, r.r)
// With x != null (k_pipe protocol) it also applies x += alpha_k p_k (p_k from pass A of this iteration)
static __global__ void __launch_bounds__(256) k_pcg_b(int64_t n, double* __restrict__ r, const double* __restrict__ Ap,
                                               const double* __restrict__ dinv, double* __restrict__ z, PcgState* st,
                                               double* partials, unsigned int* counter, double* __restrict__ x,
                                               const double* p_even, const double* p_odd) {
  __shared__ double red[32 * 3];
  if (st->stop_iter >= 0) return;
  const long long k = st->it + 1;
  const double sigma = st->red_A;
  const double rho = st->rho_hist[(k - 1) & 3];
#ifdef IPDG_DEBUG_NOBREAK  // timing builds of deliberately wrong operators (ablations): alpha = 0, no breakdown
  if (false) {
#else
  if (!(sigma > 0.0)) {  // breakdown: p^T A p <= 0 (or NaN)
#endif
    double v[2] = {0.0, 0.0}, out[2];
    if (grid_reduce<2>(v, red, partials, counter, out)) {
      st->stop_iter = k;
      st->status = -4;
      st->final_rr = st->red_B[1];
      st->it = k;
    }
    return;
  }
#ifdef IPDG_DEBUG_NOBREAK
  const double alpha = 0.0 * (rho / sigma);
#else
  const double alpha = rho / sigma;
#endif
  const double* __restrict__ p = (k & 1) ? p_odd : p_even;
  double rz = 0.0, rr = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (x) x[i] = fma(alpha, p[i], x[i]);
    const double ri = r[i] - alpha * Ap[i];
    r[i] = ri;
    const double zi = dinv ? ri * dinv[i] : ri;
    if (dinv) z[i] = zi;
    rz += ri * zi;
    rr += ri * ri;
  }
  double v[2] = {rz, rr}, out[2];
  if (grid_reduce<2>(v, red, partials, counter, out)) {
    st->red_B[0] = out[0];
    st->red_B[1] = out[1];
    st->it = k;
  }
}

// ---- PCG start: r = b - A x0, partial (r.z, r.r, b.b)
static __global__ void __launch_bounds__(256) k_pcg_init(int64_t n, const double* __restrict__ b, const double* __restrict__ Ax,
                                                  double* __restrict__ r, const double* __restrict__ dinv,
                                                  double* __restrict__ z, PcgState* st, double* partials,
                                                  unsigned int* counter) {
  __shared__ double red[32 * 3];
  double rz = 0.0, rr = 0.0, bb = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double bi = b[i];
    const double ri = bi - Ax[i];
    r[i] = ri;
    const double zi = dinv ? ri * dinv[i] : ri;
    if (dinv) z[i] = zi;
    rz += ri * zi;
    rr += ri * ri;
    bb += bi * bi;
  }
  double v[3] = {rz, rr, bb}, out[3];
  if (grid_reduce<3>(v, red, partials, counter, out)) {
    st->red_B[0] = out[0];
    st->red_B[1] = out[1];
    st->red_B[2] = out[2];
  }
}

// ---- finalize: apply the pending x += alpha_k p_k when the loop ended without a stop decision
static __global__ void __launch_bounds__(256) k_pcg_final_x(int64_t n, double* __restrict__ x, const double* p_even,
                                                     const double* p_odd, const PcgState* st) {
  if (st->stop_iter >= 0) return;
  const long long k = st->it;
  if (k < 1) return;
  const double* p = (k & 1) ? p_odd : p_even;
  const double alpha = st->rho_hist[(k - 1) & 3] / st->red_A;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] += alpha * p[i];
}
static __global__ void k_pcg_final_state(PcgState* st) {
  if (st->stop_iter >= 0) return;
  const long long k = st->it;
  st->stop_iter = k;
  const double rr = (k >= 1) ? st->red_B[1] : st->red_B[1];
  st->final_rr = rr;
  const double bb = (k >= 1) ? st->bb : st->red_B[2];
  if (k == 0) st->bb = bb;
  st->status = (rr <= st->tol2 * bb) ? 0 : 1;
}

// ---- Jacobi diagonal (setup): diag(A) per DOF from reference diagonals and geometry.
// diag_i = J [G_rr (Dr^T M Dr)_ii + 2 G_rs (Dr^T M Ds)_ii + G_ss (Ds^T M Ds)_ii] + lambda J M_ii
//        + sum over faces f containing node i (position k):
//            c_f [ -(d_n l_i, l_i)_f + tau_f (l_i, l_i)_f ],  c_f = 1 interior, 2 Dirichlet, 0 Neumann
// with (l_i,l_i)_f = sJ M1D_kk and (d_n l_i, l_i)_f = sJ (al Pr_fk + be Ps_fk),
// Pr_fk = sum_m Dr[Fmask_fm][i] M1D[m][k] (host-tabulated), al = n.grad r, be = n.grad s.
// dt layout: Krr[NP] Krs[NP] Kss[NP] Mii[NP] Pr[NF3] Ps[NF3] M1Dkk[NFP] fmask[NF3] (as doubles).
template <int N>
__global__ void k_diag(int64_t K, const double4* __restrict__ geo, const int* __restrict__ etoe,
                       const int8_t* __restrict__ bcode, const double* __restrict__ dt, double tau_c, double lambda,
                       double* __restrict__ d) {
  using T = Tr<N>;
  constexpr int NP = T::NP, NFP = T::NFP, NF3 = T::NF3;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= K * NP) return;
  const int64_t e = idx / NP;
  const int i = (int)(idx - e * NP);
  const double4 g = geo[e];
  const double rx = g.x, sx = g.y, ry = g.z, sy = g.w;
  const double J = 1.0 / (rx * sy - sx * ry);
  const double *Krr = dt, *Krs = dt + NP, *Kss = dt + 2 * NP, *Mii = dt + 3 * NP, *Pr = dt + 4 * NP, *Ps = Pr + NF3,
               *Mkk = Ps + NF3, *fm = Mkk + NFP;
  double v = J * ((rx * rx + ry * ry) * Krr[i] + 2.0 * (rx * sx + ry * sy) * Krs[i] + (sx * sx + sy * sy) * Kss[i]);
  v += lambda * J * Mii[i];
  for (int f = 0; f < 3; ++f) {
    const int bc = bcode[e * 3 + f];
    if (bc == 2) continue;
    for (int kk = 0; kk < NFP; ++kk) {
      if ((int)fm[f * NFP + kk] != i) continue;
      const double gx = (f == 0) ? -sx : (f == 1) ? rx + sx : -rx;
      const double gy = (f == 0) ? -sy : (f == 1) ? ry + sy : -ry;
      const double glen = sqrt(gx * gx + gy * gy);
      const double sJ = J * glen, nx = gx / glen, ny = gy / glen;
      double invJp = 0.0;
      if (bc == 0 || bc == 3) {
        const double4 h = geo[etoe[e * 3 + f]];
        invJp = h.x * h.w - h.y * h.z;
      }
      const double tau = tau_c * sJ * fmax(1.0 / J, invJp);
      const double al = nx * rx + ny * ry, be = nx * sx + ny * sy;
      const double dnl = sJ * (al * Pr[f * NFP + kk] + be * Ps[f * NFP + kk]);
      const double ll = sJ * Mkk[kk];
      v += (bc == 1 ? 2.0 : 1.0) * (-dnl + tau * ll);
    }
  }
  d[idx] = v;
}

// ---- block-diagonal mass and physical nodes (setup / right-hand sides)
template <int N>
__global__ void k_mass(int64_t K, const double4* __restrict__ geo, const double* __restrict__ M,
                       const double* __restrict__ u, double* __restrict__ Mu) {
  constexpr int NP = Tr<N>::NP;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= K * NP) return;
  const int64_t e = idx / NP;
  const int i = (int)(idx - e * NP);
  const double4 g = geo[e];
  const double J = 1.0 / (g.x * g.w - g.y * g.z);
  double s = 0.0;
  for (int j = 0; j < NP; ++j) s += M[i * NP + j] * u[e * NP + j];
  Mu[idx] = J * s;
}

static __global__ void k_nodes(int64_t K, int NP, const double* __restrict__ vxy, const double* __restrict__ rs,
                        double* __restrict__ x, double* __restrict__ y) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= K * NP) return;
  const int64_t e = idx / NP;
  const int i = (int)(idx - e * NP);
  const double r = rs[i], s = rs[NP + i];
  const double* v = vxy + e * 6;  // x1 y1 x2 y2 x3 y3
  x[idx] = 0.5 * (-(r + s) * v[0] + (1 + r) * v[2] + (1 + s) * v[4]);
  y[idx] = 0.5 * (-(r + s) * v[1] + (1 + r) * v[3] + (1 + s) * v[5]);
}

// ---- geometric factors from vertex coordinates (Eq. operators2): r_x = y_s/J, ... ; J <= 0 flagged
static __global__ void k_geometry(int64_t K, const double* __restrict__ vxy, double4* __restrict__ geo,
                           unsigned long long* bad) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= K) return;
  const double* v = vxy + e * 6;
  const double xr = 0.5 * (v[2] - v[0]), xs = 0.5 * (v[4] - v[0]);
  const double yr = 0.5 * (v[3] - v[1]), ys = 0.5 * (v[5] - v[1]);
  const double J = xr * ys - xs * yr;
  if (!(J > 0.0)) atomicMin(bad, (unsigned long long)e);
  geo[e] = make_double4(ys / J, -yr / J, -xs / J, xr / J);
}

}  // namespace ipdg
