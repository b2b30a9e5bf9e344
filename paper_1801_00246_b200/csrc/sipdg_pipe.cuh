// Software-pipelined fused SIPDG kernel (variant 4).  Paper: arXiv:1801.00246; formulation in
// kernels.cuh, phase structure as k_sipdg (sipdg_kernels.cuh):
//   P1  [u_r | u_s] = u [Dr^T | Ds^T] on DMMA for own + ghost tiles      (Alg. AxG)
//   P2  jump, mirrored boundary traces, central flux + penalty per own face node
//                                                                          (Alg. AxKernel)
//   P3  Au = [w_r | w_s | face block] x [Sr; Ss; LIFT^T Sr; LIFT^T Ss; E^T] on DMMA (+ lambda J M u)
// What differs from k_sipdg:
//  * Two staging buffers: the rows of block b+1 (own rows and per-element geometry records by TMA
//    bulk copies, ghost rows by cp.async) stream in while block b computes from the other buffer, so
//    the load latency of a block overlaps the previous block's DMMA work.
//  * The kernels compute from the staged rows directly.  PCG pass A forms p_k = z + beta p_{k-1}
//    where it reads an operand (P1 A fragments, P2 traces, P3 epilogue) with one fused multiply-add,
//    bit-identical everywhere; P1 also writes p_k and the deferred x update of the own rows.
//  * Geometric factors come as per-element records computed once at setup (k_geofacs): J G^T G for
//    the chain rule and, per face, the lift coefficients and sJ tau -- no divisions or square roots
//    in the hot loop.
//  * Only the face traces -sJ n.grad u (3 Nfp per slot) are kept in shared memory for the flux.
#pragma once
#include "sipdg_kernels.cuh"
#include "sipdg_split.cuh"

namespace ipdg {

template <int N>
struct TrPipe {
  using T = Tr<N>;
  static constexpr int TS = (T::NF3 + 4) | 1;   // trace row stride (odd: gathers spread over banks); columns
                                                 // NF3..NF3+3 = per-lane junk (no write-write races)
  static constexpr int OSTR = T::E * T::NP + 2;  // own staging array stride (TMA head alignment pad)
  static constexpr int GF = kGF;                 // per-face record: (c_r, c_s, sJ tau) x 3 faces (+1 pad)
  // ghost rows arrive by one bulk copy each of the 16-byte-aligned span around the row: GSTR doubles
  // (Np + 1 rounded up to even when Np is odd: the row may start on an odd double)
  static constexpr int GSTR = (T::NP & 1) ? T::NP + 1 : T::NP;
};

struct PipeLayout {
  // offsets in doubles
  int tabG, tabM, tabL, iaux, meta, trc, gid, mbar, xs, stg, sz;
  int o_u0, o_u1, o_g0, o_g1, o_gG, o_gF, o_nb, o_gs;  // within one staging buffer
  template <int N>
  // xs: PCG pass A stages x for the deferred update (else pass B updates x, see AxArgs::defer_x)
  __host__ __device__ static PipeLayout make(int gmax, bool lam, bool pcg, bool xs = true) {
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
    L.meta = o; o += 8;                       // ints: 4 x (e0, e1, g0, g1) block metadata ring
    o = (o + 1) & ~1;
    L.trc = o; o += slots * P::TS;
    L.gid = o; o += gm8;                      // 2 x gm8 ints
    o = (o + 1) & ~1;
    L.mbar = o; o += 2;
    L.xs = o; o += (pcg && xs) ? P::OSTR : 0;  // own rows of x for the deferred update (single buffer)
    // one staging buffer (two of them): own rows | p_{k-1} own | ghost rows | p_{k-1} ghosts |
    // J G^T G + J per slot | face records (own) | neighbour slots (own)
    int q = 0;
    L.o_u0 = q; q += P::OSTR;
    L.o_u1 = q; q += pcg ? P::OSTR : 0;
    L.o_g0 = q; q += gm8 * P::GSTR;
    L.o_g1 = q; q += pcg ? gm8 * P::GSTR : 0;
    q = (q + 1) & ~1;
    L.o_gG = q; q += slots * 4;
    L.o_gF = q; q += T::E * P::GF;
    L.o_nb = q; q += T::E;
    L.o_gs = q; q += gm8 / 8;                 // int8 per ghost: row start within its span (0 or 1)
    q = (q + 1) & ~1;
    L.sz = q;
    L.stg = o; o += 2 * q;
    return L;
  }
  __host__ __device__ int total() const { return stg + 2 * sz; }
};

// mbarrier transaction bookkeeping without an arrival (the arrival comes once every issuing thread
// has registered its bytes), and the plain arrival
__device__ __forceinline__ void mbar_add_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// trace columns of reference node i (row-by-row node order, refops.cpp): bits 5f..5f+4 = the column
// f*Nfp + k of the trace row when Fmask[f][k] = i, else the junk column JUNK (branch-free stores; each of
// the 4 lanes of an element row has its own junk column)
template <int N>
__host__ __device__ inline int node_trace_cols(int i, int JUNK) {
  constexpr int NFP = N + 1;
  int j = 0, off = 0;
  while (j <= N && off + (N + 1 - j) <= i) { off += N + 1 - j; ++j; }
  if (j > N) return JUNK | (JUNK << 5) | (JUNK << 10);
  const int m = i - off;
  const int c0 = (j == 0) ? m : JUNK;
  const int c1 = (m == N - j) ? NFP + j : JUNK;
  const int c2 = (m == 0) ? 2 * NFP + j : JUNK;
  return c0 | (c1 << 5) | (c2 << 10);
}

// Setup: per-element geometry records (Eq. operators2; penalty Eq. Ch2.PenaltyParameter).
//   gG[e] = (J G_rr, J G_rs, J G_ss, J), G_rr = r_x^2 + r_y^2, G_rs = r_x s_x + r_y s_y, G_ss = s_x^2 + s_y^2
//   gF[e][3f..3f+2] = (1/2 sJ n.grad r, 1/2 sJ n.grad s, sJ tau_f) with sJ n = J g_f,
//   g_f = -grad s, grad r + grad s, -grad r, and sJ tau_f = tau_c sJ^2 max(1/J, 1/J+) (1/h = sJ/J)
static __global__ void k_geofacs(int64_t K, int64_t KH, const double4* __restrict__ geo, const int* __restrict__ etoe,
                          const int8_t* __restrict__ bcode, double tau_c, double4* __restrict__ gG,
                          double* __restrict__ gF) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= KH) return;
  const double4 g = geo[e];
  const double rx = g.x, sx = g.y, ry = g.z, sy = g.w;
  const double det = rx * sy - sx * ry;
  const double J = 1.0 / det;
  gG[e] = make_double4(J * (rx * rx + ry * ry), J * (rx * sx + ry * sy), J * (sx * sx + sy * sy), J);
  if (e >= K) return;
  for (int f = 0; f < 3; ++f) {
    const double gx = (f == 0) ? -sx : (f == 1) ? rx + sx : -rx;
    const double gy = (f == 0) ? -sy : (f == 1) ? ry + sy : -ry;
    const int bc = bcode[e * 3 + f];
    double detp = 0.0;
    if (bc == 0 || bc == 3) {
      const double4 h = geo[etoe[e * 3 + f]];
      detp = h.x * h.w - h.y * h.z;
    }
    double* r = gF + e * kGF + 3 * f;
    r[0] = 0.5 * J * (rx * gx + ry * gy);
    r[1] = 0.5 * J * (sx * gx + sy * gy);
    r[2] = tau_c * (J * J * (gx * gx + gy * gy)) * fmax(det, detp);
  }
}

template <int N, int MODE, bool LAM>
__global__ void __launch_bounds__(Tr<N>::W * 32, Tr<N>::MINB) k_pipe(AxArgs a, int gmax) {
  using T = Tr<N>;
  using P = TrPipe<N>;
  constexpr int NP = T::NP, NFP = T::NFP, NT = T::NT, TS = P::TS, GF = P::GF;
  constexpr int W = T::W, E = T::E, KCG = T::KCG, KCW = T::KCW, KCM = T::KCM;
  constexpr int NTHR = W * 32;
  // bulk-copy issue duty on the last warps, which get no ghost P1 tile while Gb <= 8 (W - 2)
  constexpr int TMA_T = NTHR - 32, XTMA_T = NTHR - 64;
  constexpr bool PCG = (MODE == MODE_PCG_A);
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[32 * 3];
  const PipeLayout L = PipeLayout::make<N>(gmax, LAM, PCG, a.defer_x != 0);
  const int gm8 = (gmax + 7) / 8 * 8;
  double* tabG = sm + L.tabG;
  double* tabM = sm + L.tabM;
  double* tabL = sm + L.tabL;
  int* nidx = reinterpret_cast<int*>(sm + L.iaux);
  int* meta = reinterpret_cast<int*>(sm + L.meta);
  double* trc = sm + L.trc;
  int* gids0 = reinterpret_cast<int*>(sm + L.gid);
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(sm + L.mbar);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t K = a.K;
  const int G = gridDim.x;
  // blocks to process: all (list position = block id), or the ids in a.blist (interior / halo-boundary
  // subsets of a split pass A, overlapping the halo exchange)
  const int nbl = a.blist ? a.nlist : a.nblocks;
  auto bid = [&](int j) -> int { return a.blist ? a.blist[j] : j; };

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
  const bool with_p = PCG && !d.first;   // p_{k-1} staged: p_k = z + beta p_{k-1}
  const bool with_x = PCG && d.do_xupd && a.defer_x;  // deferred x += alpha_{k-1} p_{k-1} (else pass B updates x)
  const double beta = d.beta, alpha_prev = d.alpha_prev;

  // ---- once per CTA: operator tables, index table, metadata of the first blocks
  {
    const double* src = a.tables;
    constexpr int ntab = T::TAB_G + T::TAB_M + (LAM ? T::TAB_L : 0);  // multiple of 32 doubles
    for (int i = 2 * tid; i < ntab; i += 2 * NTHR) cp_async16(sm + i, src + i);
    for (int q = tid; q < 6 * NFP; q += NTHR) {  // nidx[fp][flip][k] = Fmask[fp][flip ? Nfp-1-k : k]
      const int fp = q / (2 * NFP), fl = (q / NFP) & 1, kk = q % NFP;
      nidx[q] = fmask_cf<N>(fp, fl ? NFP - 1 - kk : kk);
    }
    if (tid < 12) {  // metadata of this CTA's blocks 0, 1, 2 -> ring slots 0, 1, 2
      const int j = tid >> 2, w = tid & 3;
      const int b = blockIdx.x + j * G;
      int v = 0;
      if (b < nbl) v = (w < 2) ? a.boff[bid(b) + w] : a.goff[bid(b) + w - 2];
      meta[4 * j + w] = v;
    }
    for (int i = tid; i < 2 * L.sz; i += NTHR) sm[L.stg + i] = 0.0;  // padding rows stay finite
    if (tid == 0) {
      mbar_init(mbar, 1);
      mbar_init(mbar + 1, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (blockIdx.x < nbl) {  // ghost ids of block 0 (plain loads, once)
      const int g0 = meta[2], g1 = meta[3];
      for (int g = tid; g < g1 - g0; g += NTHR) gids0[g] = a.gid[g0 + g];
    }
    __syncthreads();
  }

  // ---- issue the loads of one block into staging buffer `sb`: every copy registers its bytes on
  // mbar (no arrival); thread TMA_T arrives once all threads have issued (after the next block barrier)
  auto issue = [&](double* sb, const int* mt, const int* gl, int& shift, bool& tma) {
    constexpr int GSTR = P::GSTR;
    const int64_t e0 = mt[0];
    const int Eb = mt[1] - mt[0], Gb = mt[3] - mt[2];
    double* gG = sb + L.o_gG;
    short4* nb = reinterpret_cast<short4*>(sb + L.o_nb);
    for (int e = tid; e < Eb; e += NTHR) cp_async8(nb + e, a.nbr + e0 + e);
    // own rows: one contiguous range per vector -> TMA bulk copies (16-byte aligned: the copy starts
    // one double early when the range starts on an odd double; the array's tail block falls back to
    // cp.async).  Records of 32 B / 96 B per element are always aligned.
    const int64_t g0 = e0 * NP;
    shift = (int)(g0 & 1);
    const int64_t gbase = g0 - shift;
    const unsigned nbytes = (unsigned)(((Eb * NP + shift) * 8 + 15) & ~15);
    tma = (gbase + nbytes / 8 <= K * NP);
    if (tid == TMA_T) {
      const unsigned rec = (unsigned)Eb * 32u + (unsigned)Eb * (8u * GF);
      mbar_add_tx(mbar, rec + (tma ? nbytes * (1u + (with_p ? 1u : 0u)) : 0u));
      tma_load_1d(gG, a.gG + e0, (unsigned)Eb * 32u, mbar);
      tma_load_1d(sb + L.o_gF, a.gF + e0 * GF, (unsigned)Eb * (8u * GF), mbar);
      if (tma) {
        tma_load_1d(sb + L.o_u0, U + gbase, nbytes, mbar);
        if (with_p) tma_load_1d(sb + L.o_u1, pold + gbase, nbytes, mbar);
      }
    }
    if (!tma) {
      shift = 0;
      for (int q = tid; q < Eb * NP; q += NTHR) {
        cp_async8(sb + L.o_u0 + q, U + g0 + q);
        if (with_p) cp_async8(sb + L.o_u1 + q, pold + g0 + q);
      }
    }
    double* gz = sb + L.o_g0;
    double* gp = sb + L.o_g1;
    int8_t* gs = reinterpret_cast<int8_t*>(sb + L.o_gs);
    // ghosts: records (2 x 16 B) and the 16-byte-aligned span around each row in 16-byte chunks
    for (int q = tid; q < 2 * Gb; q += NTHR) {
      const int g = q >> 1, h = q & 1;
      cp_async16(gG + (E + g) * 4 + 2 * h, reinterpret_cast<const double*>(a.gG + gl[g]) + 2 * h);
    }
    constexpr int NCH = GSTR / 2;
    for (int q = tid; q < Gb * NCH; q += NTHR) {
      const int g = q / NCH, ch = q - g * NCH;
      const int ge = gl[g];
      const bool halo = ge >= K;
      const double* base = halo ? a.halo_p : U;
      const int64_t off = (halo ? (int64_t)(ge - K) : (int64_t)ge) * NP;
      const int sh = (int)(off & 1);
      const bool span = (off - sh + GSTR) <= (halo ? a.H : K) * NP;  // the span stays inside the array
      double* dz = gz + g * GSTR;
      double* dp = gp + g * GSTR;
      if (ch == 0) gs[g] = (int8_t)(span ? sh : 0);
      if (span) {
        cp_async16(dz + 2 * ch, base + off - sh + 2 * ch);
        if (with_p) {
          if (halo) { dp[2 * ch] = 0.0; dp[2 * ch + 1] = 0.0; }  // halo rows are already p_k
          else cp_async16(dp + 2 * ch, pold + off - sh + 2 * ch);
        }
      } else {  // last row of the array: element-wise
        for (int i = 2 * ch; i < 2 * ch + 2 && i < NP; ++i) {
          cp_async8(dz + i, base + off + i);
          if (with_p) {
            if (halo) dp[i] = 0.0;
            else cp_async8(dp + i, pold + off + i);
          }
        }
      }
    }
  };

  // ---- x rows of a block for the deferred update (issued once every warp has read the previous ones)
  auto issue_x = [&](const int* mt) {
    const int64_t e0 = mt[0];
    const int Eb = mt[1] - mt[0];
    const int64_t g0 = e0 * NP;
    const int shift = (int)(g0 & 1);
    const int64_t gbase = g0 - shift;
    const unsigned nbytes = (unsigned)(((Eb * NP + shift) * 8 + 15) & ~15);
    double* xs = sm + L.xs;
    if (gbase + nbytes / 8 <= K * NP) {
      if (tid == XTMA_T) {
        mbar_expect_tx(mbar + 1, nbytes);
        tma_load_1d(xs, a.x + gbase, nbytes, mbar + 1);
      }
    } else {
      if (tid == XTMA_T) mbar_expect_tx(mbar + 1, 0u);
      for (int q = tid; q < Eb * NP; q += NTHR) cp_async8(xs + q, a.x + g0 + q);
    }
  };

  // per-lane tables: trace columns of the C-fragment nodes 8 nt + 2 (lane & 3) + h; face-node items
  // of P2 (4 lanes per element): fk = 4q + (lane & 3) -> (f, k, node); pad items repeat a real one
  // (their B rows are zero)
  int tcol[2 * NT];
#pragma unroll
  for (int q = 0; q < 2 * NT; ++q) tcol[q] = node_trace_cols<N>(8 * (q >> 1) + 2 * (lane & 3) + (q & 1), T::NF3 + (lane & 3));
  int itab[T::NQ];
#pragma unroll
  for (int q = 0; q < T::NQ; ++q) {
    const int fk = 4 * q + (lane & 3);
    const int f = fk / NFP, kk = fk - f * NFP;
    itab[q] = (fk < T::NF3) ? ((f << 24) | (kk << 16) | fmask_cf<N>(f, kk))
                            : ((2 << 24) | (N << 16) | fmask_cf<N>(2, N));
  }

  int cur_shift = 0, nxt_shift = 0;
  bool cur_tma = false, nxt_tma = false;
  if (blockIdx.x < nbl) {
    issue(sm + L.stg, meta, gids0, cur_shift, cur_tma);
    if (with_x) issue_x(meta);
    __syncthreads();  // every thread has registered its copies
    if (tid == TMA_T) mbar_arrive(mbar);
    const int b1 = blockIdx.x + G;
    if (b1 < nbl) {  // ghost ids of block 1 -> gids[1]
      const int g0 = meta[4 + 2], g1 = meta[4 + 3];
      for (int g = tid; g < g1 - g0; g += NTHR) cp_async4(gids0 + gm8 + g, a.gid + g0 + g);
    }
  }
  cp_async_commit();

  unsigned phase = 0, xphase = 0;
#ifdef IPDG_PHASE_TIMING
  long long ph_t = clock64();
#endif
  double wr[NT][2], ws[NT][2];
  int it = 0;
  for (int b = blockIdx.x; b < nbl; b += G, ++it) {
    const int par = it & 1;
    const int* mt = meta + 4 * (it & 3);
    const int64_t e0 = mt[0];
    const int Eb = mt[1] - mt[0], Gb = mt[3] - mt[2];
    double* sb = sm + L.stg + par * L.sz;
    // operand rows of this block: own slot s < E at su[s*NP], ghost slot E+g at sg[g*NP] (+ p_{k-1})
    const double* su = sb + L.o_u0 + cur_shift;
    const double* sp = sb + L.o_u1 + cur_shift;
    const double* sg = sb + L.o_g0;
    const double* sgp = sb + L.o_g1;
    const int8_t* gsh = reinterpret_cast<const int8_t*>(sb + L.o_gs);
    const double* gGs = sb + L.o_gG;
    const double* gFs = sb + L.o_gF;
    const short4* nbs = reinterpret_cast<const short4*>(sb + L.o_nb);
    // ---- wait for this block's staged data (issued one block earlier)
    cp_async_wait_all();
    mbar_wait(mbar, phase);
    phase ^= 1u;
    if (with_x) {
      mbar_wait(mbar + 1, xphase);
      xphase ^= 1u;
    }
    __syncthreads();  // also: every warp is done with the other buffer (block b - G)
    PHASE_MARK(0);  // wait for this block's data
    // ---- issue block b + G into the other buffer, ghost ids of block b + 2G, metadata of b + 3G
    {
      const int b1 = b + G, b2 = b + 2 * G, b3 = b + 3 * G;
      if (b1 < nbl)
        issue(sm + L.stg + (par ^ 1) * L.sz, meta + 4 * ((it + 1) & 3), gids0 + (par ^ 1) * gm8, nxt_shift, nxt_tma);
      if (b2 < nbl) {
        const int* m2 = meta + 4 * ((it + 2) & 3);
        const int g0 = m2[2], g1 = m2[3];
        int* gdst = gids0 + par * gm8;
        for (int g = tid; g < g1 - g0; g += NTHR) cp_async4(gdst + g, a.gid + g0 + g);
      }
      if (tid < 4 && b3 < nbl) {
        int* m3 = meta + 4 * ((it + 3) & 3);
        const int b3i = bid(b3);
        if (tid < 2) cp_async4(m3 + tid, a.boff + b3i + tid);
        else cp_async4(m3 + tid, a.goff + b3i + tid - 2);
      }
      cp_async_commit();
    }
    PHASE_MARK(1);  // issue of the next block's loads
    if (PCG) {  // form p_k = z + beta p_{k-1} in place (own + ghost rows); own rows also write p_k
      // and apply the deferred x update x += alpha_{k-1} p_{k-1} (coalesced)
      double* wu = sb + L.o_u0 + cur_shift;
      const double* xs = sm + L.xs + cur_shift;
      for (int q = tid; q < Eb * NP; q += NTHR) {
        const double po = with_p ? sp[q] : 0.0;
        const double v = with_p ? fma(beta, po, wu[q]) : wu[q];
        const int64_t g = e0 * NP + q;
        wu[q] = v;
        pnew[g] = v;
        if (with_x) a.x[g] = fma(alpha_prev, po, xs[q]);
      }
      if (with_p) {
        double* wg = sb + L.o_g0;
        for (int q = tid; q < Gb * NP; q += NTHR) {
          const int g = q / NP, i = q - g * NP;
          const int o = g * P::GSTR + gsh[g] + i;
          wg[o] = fma(beta, sgp[o], wg[o]);
        }
      }
      __syncthreads();
    }
    // operand value at slot s, node i (PCG: p_k, formed above)
    auto uval = [&](int s, int i) -> double {
      if (s < E) return su[s * NP + i];
      return sg[(s - E) * P::GSTR + gsh[s - E] + i];
    };
    PHASE_MARK(2);  // PCG: p_k and x stores
    // ---- P1: reference gradient on DMMA; face traces to smem; w_r / w_s kept in registers (own)
    const int ntiles = W + (Gb + 7) / 8;
    for (int t = warp; t < ntiles; t += W) {
      const bool own = t < W;
      const int sbase = own ? 8 * t : E + 8 * (t - W);
      if (own && sbase >= Eb) continue;
      const int srow = sbase + (lane >> 2);
      double av[KCG];
#pragma unroll
      for (int kc = 0; kc < KCG; ++kc) {
        const int i = 4 * kc + (lane & 3);
        av[kc] = (i < NP) ? uval(srow, i) : 0.0;
      }
      double acc[2 * NT][2];
#pragma unroll
      for (int q = 0; q < 2 * NT; ++q) acc[q][0] = acc[q][1] = 0.0;
#pragma unroll
      for (int kc = 0; kc < KCG; ++kc) {
        const double* bt = tabG + kc * 2 * NT * 32 + lane;
#pragma unroll
        for (int q = 0; q < 2 * NT; ++q) dmma(acc[q][0], acc[q][1], av[kc], bt[q * 32]);
      }
      // w_r = J (G_rr u_r + G_rs u_s), w_s = J (G_rs u_r + G_ss u_s); the scaled normal derivatives
      // sJ n.grad u on faces 0, 1, 2 are -w_s, w_r + w_s, -w_r (J g_f.grad u, g_f = -grad s,
      // grad r + grad s, -grad r)
      const double* gq = gGs + srow * 4;
      const double Grr = gq[0], Grs = gq[1], Gss = gq[2];
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
    PHASE_MARK(3);  // P1 + volume DMMAs (warp 0)
    __syncthreads();  // traces of every slot written; x rows of this block consumed
    PHASE_MARK(4);  // barrier
    if (tid == TMA_T && b + G < nbl) mbar_arrive(mbar);  // block b + G: every copy is registered
    if (with_x && b + G < nbl) issue_x(meta + 4 * ((it + 1) & 3));

    // ---- P2 + P3 face part per warp on its own tile
    if (8 * warp < Eb) {
      const int ec = e < Eb ? e : 8 * warp;  // rows past the block end compute on a valid slot, never stored
      const short4 nb = nbs[ec];
      const double* to = trc + ec * TS;
      const double* fq0 = gFs + ec * GF;
#pragma unroll
      for (int q = 0; q < T::NQ; ++q) {
        const int itq = itab[q];
        const int f = itq >> 24, kk = (itq >> 16) & 255, i = itq & 65535;
        const int fl = (nb.w >> (4 * f)) & 15;
        const int fp = fl & 3, bc = fl >> 2;
        const int slot = (f == 0) ? nb.x : (f == 1) ? nb.y : nb.z;
        const double* fq = fq0 + 3 * f;
        // boundary faces read the element's own trace and mirror it (R7):
        // Dirichlet u+ = -u-, grad u+ = grad u-;  Neumann u+ = u-, grad u+ = -grad u-
        const bool inner = (bc == 0);
        const int flip = inner && ((f == 2) == (fp == 2));
        const int ps = inner ? slot : ec;
        const int kq = flip ? NFP - 1 - kk : kk;
        const int tpi = inner ? fp * NFP + kq : f * NFP + kk;
        const int ip = inner ? nidx[(2 * fp + flip) * NFP + kk] : i;
        const double um = uval(ec, i), upr = uval(ps, ip);
        const double tm = to[f * NFP + kk];     // -sJ n-.grad u-
        const double tp = trc[ps * TS + tpi];   // -sJ n+.grad u+ (the neighbour's own normal)
        const double delta = ((bc == 1) ? -upr : upr) - um;     // paper jump
        const double far = fq[0] * delta;                       // 1/2 sJ (n.grad r) delta
        const double fas = fq[1] * delta;                       // 1/2 sJ (n.grad s) delta
        // -sJ (n-.{grad u} + tau delta); n-.grad u+ = -n+.grad u+ inside, = n-.grad u- mirrored on Dirichlet
        const double hp = (bc == 1) ? 0.5 : -0.5;
        const double fag = fma(0.5, tm, fma(hp, tp, -fq[2] * delta));
        const double* b0 = tabM + (KCW + q) * NT * 32 + lane;
        const double* b1 = tabM + (KCW + T::NQ + q) * NT * 32 + lane;
        const double* b2 = tabM + (KCW + 2 * T::NQ + q) * NT * 32 + lane;
        // chains interleaved: consecutive DMMAs go to different accumulators (26.6-cycle DMMA latency)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(C[j][0], C[j][1], far, b0[j * 32]);
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(C[j][0], C[j][1], fas, b1[j * 32]);
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(C[j][0], C[j][1], fag, b2[j * 32]);
      }
      if (LAM) {
        const double lj = a.lambda * gGs[ec * 4 + 3];
#pragma unroll
        for (int kc = 0; kc < KCM; ++kc) {
          const int i = 4 * kc + (lane & 3);
          const double av = (i < NP) ? lj * uval(ec, i) : 0.0;
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
              if (PCG) dot += uval(e, i) * C[nt][h];
            }
          }
      }
    }
    PHASE_MARK(5);  // P2 + P3 faces + stores (warp 0)
    cur_shift = nxt_shift;
    cur_tma = nxt_tma;
  }
  cp_async_wait_all();
  if (PCG) {
    double v[1] = {dot}, out[1];
    if (grid_reduce<1>(v, red, a.partials, a.counter, out)) {
      PcgState* st = a.st;
      // split pass A: the first launch parks its partial p.Ap, the second adds it (red_A is still read
      // as alpha_{k-1}'s denominator by the second launch's prologue)
      if (a.red_part == 1) st->red_A_part = out[0];
      else st->red_A = (a.red_part == 2) ? st->red_A_part + out[0] : out[0];
      st->rho_hist[(d.k - 1) & 3] = d.rhoB;
      if (d.first) st->bb = d.bbv;
    }
  }
}

}  // namespace ipdg
