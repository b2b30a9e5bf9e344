// Per-degree host dispatch (Impl<N>): fragment tables, launch configuration, variant choice and the
// kernel launches of Ax / PCG pass A / block-Jacobi / DG operators.  Included by impl_N.cu only, so the
// N = 1..8 kernel instantiations compile as separate translation units in parallel.
// Paper: arXiv:1801.00246 (P:n = PAPER.md line n).
#pragma once
#include "ctx.h"
#include "sipdg_kernels.cuh"
#include "sipdg_split.cuh"
#include "sipdg_pipe.cuh"
#include "pcg_blockjacobi.cuh"
#include "cops.cuh"
#include "sipdg_gather.cuh"
#include "dgops.cuh"
#include "sipdg_tpb.cuh"
#include "advect.cuh"

#ifndef IPDG_TPB_MAXN
#define IPDG_TPB_MAXN 8  // highest degree with a k_tpb instantiation (lower it for quick rebuilds)
#endif

// ------------------------------------------------------------------ per-N dispatch
template <int N>
struct Impl {
  using T = Tr<N>;

  // DMMA fragment tables: [chunk][ntile][lane], lane -> (k = lane & 3, n = lane >> 2)
  static std::vector<double> build_tables(const RefOps& R) {
    const int NP = T::NP, NFP = T::NFP, NF3 = T::NF3, NT = T::NT;
    std::vector<double> tab(T::TAB_G + T::TAB_M + T::TAB_L, 0.0);
    double* tg = tab.data();
    double* tm = tg + T::TAB_G;
    double* tl = tm + T::TAB_M;
    auto at = [&](const std::vector<double>& A, int ld, int i, int j, int ni, int nj) {
      return (i < ni && j < nj) ? A[i * ld + j] : 0.0;
    };
    for (int kc = 0; kc < T::KCG; ++kc)
      for (int q = 0; q < 2 * NT; ++q)
        for (int l = 0; l < 32; ++l) {
          const int k = 4 * kc + (l & 3), n = 8 * (q % NT) + (l >> 2);
          const std::vector<double>& D = (q < NT) ? R.Dr : R.Ds;
          tg[(kc * 2 * NT + q) * 32 + l] = at(D, NP, n, k, NP, NP);  // B[k][n] = D[n][k]
        }
    // LIFT^T Sr, LIFT^T Ss  (3Nfp x Np)
    std::vector<double> LSr(NF3 * NP, 0.0), LSs(NF3 * NP, 0.0);
    for (int m = 0; m < NF3; ++m)
      for (int n = 0; n < NP; ++n) {
        double a = 0, b = 0;
        for (int i = 0; i < NP; ++i) {
          a += R.LIFT[i * NF3 + m] * R.Sr[i * NP + n];
          b += R.LIFT[i * NF3 + m] * R.Ss[i * NP + n];
        }
        LSr[m * NP + n] = a;
        LSs[m * NP + n] = b;
      }
    for (int c = 0; c < T::KCW + T::KCF; ++c)
      for (int j = 0; j < NT; ++j)
        for (int l = 0; l < 32; ++l) {
          const int n = 8 * j + (l >> 2);
          double v = 0.0;
          if (c < 4 * NT) {  // w_r / w_s chunks straight from the C-fragment layout
            const int cc = c % (2 * NT);
            const int i = 8 * (cc >> 1) + 2 * (l & 3) + (cc & 1);
            v = at(c < 2 * NT ? R.Sr : R.Ss, NP, i, n, NP, NP);
          } else {
            const int m = 4 * (c - 4 * NT) + (l & 3);
            const int blk = m / T::NF3P, mm = m % T::NF3P;  // three face sub-blocks, each padded to NF3P
            if (mm >= NF3) v = 0.0;
            else if (blk == 0) v = at(LSr, NP, mm, n, NF3, NP);
            else if (blk == 1) v = at(LSs, NP, mm, n, NF3, NP);
            else {  // face mass scattered to the face rows: E[n][m'] (E = M LIFT)
              const int f = mm / NFP, kk = mm % NFP;
              if (n < NP)
                for (int q = 0; q < NFP; ++q)
                  if (R.Fmask[f * NFP + q] == n) v = R.M1D[q * NFP + kk];
            }
          }
          tm[(c * NT + j) * 32 + l] = v;
        }
    for (int kc = 0; kc < T::KCM; ++kc)
      for (int j = 0; j < NT; ++j)
        for (int l = 0; l < 32; ++l) {
          const int k = 4 * kc + (l & 3), n = 8 * j + (l >> 2);
          tl[(kc * NT + j) * 32 + l] = at(R.M, NP, k, n, NP, NP);
        }
    // aux: M1D, then ints fmask[NF3], nodeface[2*NPN]
    for (int i = 0; i < NFP * NFP; ++i) tab.push_back(R.M1D[i]);
    std::vector<int> ia(NF3 + 2 * T::NPN, -1);
    for (int i = 0; i < NF3; ++i) ia[i] = R.Fmask[i];
    for (int f = 0; f < 3; ++f)
      for (int k = 0; k < NFP; ++k) {
        const int i = R.Fmask[f * NFP + k];
        int* slot = &ia[NF3 + 2 * i];
        if (slot[0] < 0) slot[0] = f * NFP + k;
        else slot[1] = f * NFP + k;
      }
    if (ia.size() % 2) ia.push_back(-1);
    const size_t base = tab.size();
    tab.resize(base + ia.size() / 2);
    std::memcpy(tab.data() + base, ia.data(), ia.size() * sizeof(int));
    // split variant (k_flux): main table with w_r, w_s rows in natural node order
    using S = TrS<N>;
    tab.resize(S::OFF_M2, 0.0);
    tm = tab.data() + T::TAB_G;  // the vector may have moved
    std::vector<double> m2(S::TAB_M2, 0.0);
    for (int c = 0; c < S::KCW2 + T::KCF; ++c)
      for (int j = 0; j < NT; ++j)
        for (int l = 0; l < 32; ++l) {
          const int n = 8 * j + (l >> 2);
          double v;
          if (c < S::KCW2) {
            const int k = 4 * (c % T::KCG) + (l & 3);
            v = at(c < T::KCG ? R.Sr : R.Ss, NP, k, n, NP, NP);
          } else {
            v = tm[((c - S::KCW2 + T::KCW) * NT + j) * 32 + l];  // face chunks: same as the fused table
          }
          m2[(c * NT + j) * 32 + l] = v;
        }
    tab.insert(tab.end(), m2.begin(), m2.end());
    return tab;
  }

  static std::vector<double> build_diagtab(const RefOps& R) {
    const int NP = T::NP, NFP = T::NFP, NF3 = T::NF3;
    std::vector<double> d(4 * NP + 2 * NF3 + NFP + NF3, 0.0);
    for (int i = 0; i < NP; ++i) {
      double krr = 0, krs = 0, kss = 0;
      for (int a = 0; a < NP; ++a)
        for (int b = 0; b < NP; ++b) {
          const double m = R.M[a * NP + b];
          krr += R.Dr[a * NP + i] * m * R.Dr[b * NP + i];
          krs += R.Dr[a * NP + i] * m * R.Ds[b * NP + i];
          kss += R.Ds[a * NP + i] * m * R.Ds[b * NP + i];
        }
      d[i] = krr;
      d[NP + i] = krs;
      d[2 * NP + i] = kss;
      d[3 * NP + i] = R.M[i * NP + i];
    }
    for (int f = 0; f < 3; ++f)
      for (int k = 0; k < NFP; ++k) {
        const int i = R.Fmask[f * NFP + k];
        double pr = 0, ps = 0;
        for (int m = 0; m < NFP; ++m) {
          const int fm = R.Fmask[f * NFP + m];
          pr += R.Dr[fm * NP + i] * R.M1D[m * NFP + k];
          ps += R.Ds[fm * NP + i] * R.M1D[m * NFP + k];
        }
        d[4 * NP + f * NFP + k] = pr;
        d[4 * NP + NF3 + f * NFP + k] = ps;
      }
    for (int k = 0; k < NFP; ++k) d[4 * NP + 2 * NF3 + k] = R.M1D[k * NFP + k];
    for (int i = 0; i < NF3; ++i) d[4 * NP + 2 * NF3 + NFP + i] = R.Fmask[i];
    return d;
  }

  static int configure(ipdg_ctx c) {
    int optin = 0;
    CUDA_TRY(c, cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
    for (int lam = 0; lam < 2; ++lam) {
      for (int mode = 0; mode < 2; ++mode) {
        const SmemLayout L = SmemLayout::make<N>(c->gmax, lam != 0, mode == 1);
        const size_t bytes = (size_t)L.total * sizeof(double);
        c->smem[mode][lam] = bytes;
        const void* fn = (mode == 0) ? (lam ? (const void*)k_sipdg<N, MODE_AX, true> : (const void*)k_sipdg<N, MODE_AX, false>)
                                     : (lam ? (const void*)k_sipdg<N, MODE_PCG_A, true>
                                            : (const void*)k_sipdg<N, MODE_PCG_A, false>);
        // opt in to the full per-CTA maximum once: the attribute is per function (shared by all
        // contexts of this N), the launch passes the context's own byte count
        if ((int)bytes > optin - 1024) FAIL(c, IPDG_ECUDA, "k_sipdg<N=%d> needs %zu B of shared memory", N, bytes);
        CUDA_TRY(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024));
        int occ = 0;
        CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, T::W * 32, bytes));
        if (occ < 1) FAIL(c, IPDG_ECUDA, "k_sipdg<N=%d> does not fit on an SM (smem %zu B, gmax %d)", N, bytes, c->gmax);
        c->grid[mode][lam] = (int)std::min<int64_t>(c->nblocks, (int64_t)occ * c->sms);
      }
    }
    // split variant
    using S = TrS<N>;
    {
      const size_t bytes = (size_t)(T::TAB_G + S::W * 8 * T::SU) * sizeof(double);
      c->smem_grad = bytes;
      const void* fns[2] = {(const void*)k_grad<N, MODE_AX>, (const void*)k_grad<N, MODE_PCG_A>};
      int occ = 1;
      for (const void* fn : fns) {
        CUDA_TRY(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024));
        int o = 0;
        CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, S::W * 32, bytes));
        occ = std::max(1, o);
      }
      const int64_t tiles = (c->K + c->H + 7) / 8;
      c->grid_grad = (int)std::max<int64_t>(1, std::min<int64_t>((tiles + S::W - 1) / S::W, (int64_t)occ * c->sms));
    }
    for (int lam = 0; lam < 2; ++lam) {
      const size_t bytes = (size_t)(S::TAB_M2 + (lam ? T::TAB_L : 0)) * sizeof(double);
      c->smem_flux[lam] = bytes;
      for (int mode = 0; mode < 2; ++mode) {
        const void* fn = (mode == 0) ? (lam ? (const void*)k_flux<N, MODE_AX, true> : (const void*)k_flux<N, MODE_AX, false>)
                                     : (lam ? (const void*)k_flux<N, MODE_PCG_A, true> : (const void*)k_flux<N, MODE_PCG_A, false>);
        CUDA_TRY(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024));
        int o = 0;
        CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, S::W * 32, bytes));
        const int64_t tiles = (c->K + 7) / 8;
        c->grid_flux[mode][lam] = (int)std::max<int64_t>(1, std::min<int64_t>((tiles + S::W - 1) / S::W, (int64_t)std::max(1, o) * c->sms));
      }
    }
    TRY(configure_tpb(c, optin));
    return configure_pipe(c, optin);
  }

  static int configure_tpb(ipdg_ctx c, int optin) {
    if constexpr (N <= IPDG_TPB_MAXN) {
    for (int lam = 0; lam < 2; ++lam)
      for (int mode = 0; mode < 2; ++mode) {
        const size_t bytes = (size_t)TpbLayout<N>::total(c->gmax_t, mode == 1) * sizeof(double);
        c->smem_tpb_m[mode] = bytes;
        const void* fn = (mode == 0) ? (lam ? (const void*)k_tpb<N, MODE_AX, true> : (const void*)k_tpb<N, MODE_AX, false>)
                                     : (lam ? (const void*)k_tpb<N, MODE_PCG_A, true> : (const void*)k_tpb<N, MODE_PCG_A, false>);
        c->tpb_ok[mode][lam] = false;
        if ((int)bytes > optin - 1024) continue;
        CUDA_TRY(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024));
        int occ = 0;
        CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, TrB<N>::NTHR, bytes));
        c->tpb_ok[mode][lam] = occ > 0;
        // persistent pass A (profiles/r02b_tpb_experiments.txt); IPDG_TPB_PERSIST=0 (measurement): one CTA
        // per block
        const char* ev = getenv("IPDG_TPB_PERSIST");
        const bool persist = ev ? atoi(ev) != 0 : true;
        // IPDG_TPB_CTAS=k (measurement): at most k resident CTAs per SM in the persistent grid
        const char* ek = getenv("IPDG_TPB_CTAS");
        const int cps = (ek && atoi(ek) > 0) ? std::min(std::max(1, occ), atoi(ek)) : std::max(1, occ);
        c->tpb_grid[mode][lam] = persist ? cps * c->sms : (1 << 30);
      }
    }
    return IPDG_OK;
  }

  // one CTA per block of tpb_e(N) elements (all blocks, or the interior / boundary lists of a split pass A)
  template <int MODE>
  static int launch_tpb(ipdg_ctx c, AxArgs& a, bool lam, cudaStream_t s, const int* list, int n, bool comm_slots = false) {
    if constexpr (N > IPDG_TPB_MAXN) {
      FAIL(c, IPDG_EINVAL, "k_tpb not built for N = %d", N);
    } else {
    a.nbt = c->nbt;
    a.gfoff = c->gfoff_t;
    a.gface = c->gface_t;
    a.tauF = c->tauF;
    a.blist = list;
    a.nlist = n;
    int grid = list ? n : c->nblocks_t;
    if (grid <= 0) return IPDG_OK;
    if (MODE == MODE_PCG_A) {  // Ax: one CTA per block
      const int pg = c->tpb_grid[1][lam ? 1 : 0];
      // while a halo exchange is in flight leave a few CTA slots free for NCCL's kernel (as k_pipe)
      grid = std::min(grid, comm_slots ? std::max(1, std::min(pg, c->sms * 4) - kCommSlots) : pg);
    }
    if (MODE == MODE_PCG_A && c->grid_cap > 0) grid = std::min(grid, c->grid_cap);
    if (MODE == MODE_PCG_A && grid > c->partials_cap) FAIL(c, IPDG_ECUDA, "partials buffer too small");
    const size_t smb = c->smem_tpb_m[MODE == MODE_PCG_A ? 1 : 0];
    if (lam) k_tpb<N, MODE, true><<<grid, TrB<N>::NTHR, smb, s>>>(a, c->gmax_t);
    else k_tpb<N, MODE, false><<<grid, TrB<N>::NTHR, smb, s>>>(a, c->gmax_t);
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    return IPDG_OK;
    }
  }

  // ---- pipelined fused variant: needs room for the staging area next to the working rows
  static int configure_pipe(ipdg_ctx c, int optin) {
    for (int lam = 0; lam < 2; ++lam)
      for (int mode = 0; mode < 2; ++mode) {
        const void* fn = (mode == 0) ? (lam ? (const void*)k_pipe<N, MODE_AX, true> : (const void*)k_pipe<N, MODE_AX, false>)
                                     : (lam ? (const void*)k_pipe<N, MODE_PCG_A, true> : (const void*)k_pipe<N, MODE_PCG_A, false>);
        c->grid_pipe[mode][lam] = 0;
        c->pipe_xb[lam] = false;
        int best = 0;
        // PCG pass A: stage x for the deferred update unless that costs a resident CTA per SM, in which
        // case pass B updates x (AxArgs::defer_x = 0)
        for (int xs = 1; xs >= (mode == 1 ? 0 : 1); --xs) {
          const PipeLayout L = PipeLayout::make<N>(c->gmax, lam != 0, mode == 1, xs != 0);
          const size_t bytes = (size_t)L.total() * sizeof(double);
          if ((int)bytes > optin - 1024) continue;
          CUDA_TRY(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024));
          int occ = 0;
          CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, T::W * 32, bytes));
          if (occ > best) {
            best = occ;
            c->smem_pipe[mode][lam] = bytes;
            c->grid_pipe[mode][lam] = (int)std::min<int64_t>(c->nblocks, (int64_t)occ * c->sms);
            if (mode == 1) c->pipe_xb[lam] = (xs == 0);
          }
        }
      }
    return IPDG_OK;
  }

  // k_tpb operator tables (sipdg_tpb.cuh): face-restricted derivative split checked against Dr / Ds
  static int upload_tpb_constants(ipdg_ctx c) {
    using B = TrB<N>;
    const RefOps& R = c->ref;
    const int NP = B::NP, NFP = B::NFP;
    std::vector<double> h(B::TOTAL, 0.0);
    auto D = [&](const std::vector<double>& A, int i, int j) { return A[i * NP + j]; };
    if constexpr (B::GRAD) {
      for (int i = 0; i < NP; ++i)
        for (int j = 0; j < NP; ++j) {
          h[B::O_DRT + j * NP + i] = D(R.Dr, i, j);
          h[B::O_DST + j * NP + i] = D(R.Ds, i, j);
          h[B::O_SR + i * NP + j] = D(R.Sr, i, j);
          h[B::O_SS + i * NP + j] = D(R.Ss, i, j);
        }
    }
    // K_rr = Dr^T M Dr, K_rs = Dr^T M Ds + Ds^T M Dr, K_ss = Ds^T M Ds (Sr = M Dr, Ss = M Ds); [j][n], symmetric
    for (int i = 0; i < NP && !B::GRAD; ++i)
      for (int j = 0; j < NP; ++j) {
        double rr = 0, rs = 0, ss = 0;
        for (int a = 0; a < NP; ++a) {
          rr += D(R.Dr, a, i) * D(R.Sr, a, j);
          rs += D(R.Dr, a, i) * D(R.Ss, a, j) + D(R.Ds, a, i) * D(R.Sr, a, j);
          ss += D(R.Ds, a, i) * D(R.Ss, a, j);
        }
        h[B::O_KRR + i * NP + j] = rr;
        h[B::O_KRS + i * NP + j] = rs;
        h[B::O_KSS + i * NP + j] = ss;
      }
    // tangential derivative d/dxi along each face (face node order) and the transverse rows T_f
    std::vector<double> D1D(NFP * NFP), Tf(3 * NFP * NP);
    for (int k = 0; k < NFP; ++k)
      for (int m = 0; m < NFP; ++m) D1D[k * NFP + m] = D(R.Dr, R.Fmask[k], R.Fmask[m]);
    double dmax = 0.0, bad = 0.0;
    for (double v : R.Dr) dmax = std::max(dmax, std::fabs(v));
    for (int f = 0; f < 3; ++f)
      for (int k = 0; k < NFP; ++k) {
        const int i = R.Fmask[f * NFP + k];
        for (int j = 0; j < NP; ++j) {
          const double tang = (f == 0) ? D(R.Dr, i, j) : (f == 1) ? D(R.Ds, i, j) - D(R.Dr, i, j) : D(R.Ds, i, j);
          double want = 0.0;
          for (int m = 0; m < NFP; ++m)
            if (R.Fmask[f * NFP + m] == j) want = D1D[k * NFP + m];
          bad = std::max(bad, std::fabs(tang - want));
          Tf[(f * NFP + k) * NP + j] = (f == 0) ? D(R.Ds, i, j) : D(R.Dr, i, j);
          h[B::O_TN + (f * NFP + k) * NP + j] = Tf[(f * NFP + k) * NP + j];
        }
      }
    if (bad > 1e-9 * dmax) FAIL(c, IPDG_ECUDA, "k_tpb: face-tangential derivative check failed (%g)", bad);
    if constexpr (!B::BIG) {
      for (int f = 0; f < 3; ++f)
        for (int n = 0; n < NP; ++n)
          for (int k = 0; k < NFP; ++k) {
            double v = 0;
            for (int m = 0; m < NFP; ++m) v += Tf[(f * NFP + m) * NP + n] * R.M1D[m * NFP + k];
            h[B::O_PT + (f * NFP + k) * NP + n] = v;
          }
      for (int m = 0; m < NFP; ++m)
        for (int k = 0; k < NFP; ++k) {
          double v = 0;
          for (int j = 0; j < NFP; ++j) v += D1D[j * NFP + m] * R.M1D[j * NFP + k];
          h[B::O_QT + k * NFP + m] = v;
        }
      for (int i = 0; i < NP * NP; ++i) h[B::O_M + i] = R.M[i];
    }
    for (int m = 0; m < NFP; ++m)
      for (int k = 0; k < NFP; ++k) {
        h[B::O_M1D + m * NFP + k] = R.M1D[m * NFP + k];
        h[B::O_D1DT + m * NFP + k] = D1D[k * NFP + m];
      }
    CUDA_TRY(c, cudaMemcpyToSymbol(c_tpb<N>, h.data(), h.size() * sizeof(double)));
    return IPDG_OK;
  }

  static int upload_constants(ipdg_ctx c) {
    TRY(upload_tpb_constants(c));
    if constexpr (N <= 4) {
      using TT = TrT<N>;
      const RefOps& R = c->ref;
      const int NP = TT::NP, NFP = TT::NFP, NF3 = TT::NF3;
      std::vector<double> h(TT::TOTAL, 0.0);
      for (int i = 0; i < NP * NP; ++i) {
        h[TT::O_DR + i] = R.Dr[i];
        h[TT::O_DS + i] = R.Ds[i];
        h[TT::O_SR + i] = R.Sr[i];
        h[TT::O_SS + i] = R.Ss[i];
        h[TT::O_M + i] = R.M[i];
      }
      for (int m = 0; m < NF3; ++m)
        for (int n = 0; n < NP; ++n) {
          double a = 0, b = 0;
          for (int i = 0; i < NP; ++i) {
            a += R.LIFT[i * NF3 + m] * R.Sr[i * NP + n];
            b += R.LIFT[i * NF3 + m] * R.Ss[i * NP + n];
          }
          h[TT::O_LSR + m * NP + n] = a;
          h[TT::O_LSS + m * NP + n] = b;
        }
      for (int i = 0; i < NFP * NFP; ++i) h[TT::O_M1D + i] = R.M1D[i];
      for (int i = 0; i < NP * NF3; ++i) h[TT::O_LIFT + i] = R.LIFT[i];
      CUDA_TRY(c, cudaMemcpyToSymbol(c_tpe<N>, h.data(), h.size() * sizeof(double)));
    }
    return IPDG_OK;
  }

  // k_pipe moves whole rows with TMA bulk copies: operand vectors must be 16-byte aligned
  static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }
  // Kernel actually used (1 fused k_sipdg, 2 split, 4 pipelined k_pipe, 5 gather, 6 thread-per-element
  // block k_tpb).  Auto (variant 0), the fastest measured per degree (profiles/r02_variants_tpb_vs_pipe.jsonl,
  // C3 and C2): k_tpb for N <= 5 (Ax and PCG pass A) except PCG pass A at N = 4, where k_pipe is 2 % faster
  // on the bench mesh C2 (76.6 vs 78.1 us; C3: 320 vs 307 us), split for N >= 6 (k_tpb's register-resident
  // rows spill there).
  // k_pipe falls back to k_sipdg when it does not fit on an SM or the operand is not 16-byte aligned.
  static int resolve(ipdg_ctx c, int mode, bool lam, const void* v) {
    int k = c->variant;
    // measured fastest per degree and pass (profiles/r02c_variants.jsonl, r02c_variants_hi.jsonl): k_tpb for
    // N <= 5; Ax at N = 6 on k_pipe (C3 657 vs 695 us for the split pair), the split pair otherwise
    if (k == 0) k = (N >= 6) ? ((mode == 0 && N == 6) ? 4 : 2) : 6;
    if (k == 3) k = 1;  // (the thread-per-element variant was retired; it was never the fastest)
    if (k == 5 && N > 4) k = 1;
    if (k == 6 && !(c->tpb_ok[mode][lam] && (!lam || TrB<N>::HAS_LAM) && (v == nullptr || aligned16(v)))) k = 1;
    if (k == 4 && !(c->grid_pipe[mode][lam] > 0 && aligned16(v))) k = 1;
    return k;
  }

  // gather variant (N <= 4): one thread per element, grid-stride
  template <int MODE>
  static int launch_gather(ipdg_ctx c, AxArgs& a, bool lam, cudaStream_t s) {
    if constexpr (N <= 4) {
      const int grid = (int)std::max<int64_t>(1, (c->K + kGatherThreads - 1) / kGatherThreads);  // one element per thread
      if (MODE == MODE_PCG_A && grid > c->partials_cap) FAIL(c, IPDG_ECUDA, "partials buffer too small");
      if (lam) k_gather<N, MODE, true><<<grid, kGatherThreads, 0, s>>>(a);
      else k_gather<N, MODE, false><<<grid, kGatherThreads, 0, s>>>(a);
      c->launches++;
      CUDA_TRY(c, cudaGetLastError());
      return IPDG_OK;
    } else {
      FAIL(c, IPDG_EINVAL, "gather variant needs N <= 4");
    }
  }

  static SplitArgs sargs(ipdg_ctx c) {
    SplitArgs a;
    std::memset(&a, 0, sizeof(a));
    a.K = c->K;
    a.H = c->H;
    a.geo = c->geo;
    a.nbg = c->nbg;
    a.tables = c->tables;
    a.tau_c = c->tau_c;
    a.halo = c->halobuf;
    a.W2 = c->W2;
    a.gG = c->gG;
    a.gF = c->gF;
    a.ebeg = 0;
    a.eend = c->K + c->H;
    a.stop_work = 1;
    return a;
  }

  // k_grad over [K, K + H) alone: the halo rows, once the exchange has landed
  static int grad_launch(ipdg_ctx c, SplitArgs a, int mode, int64_t ebeg, int64_t eend, int stop_work, cudaStream_t s,
                         int spare = 0) {
    using S = TrS<N>;
    a.ebeg = ebeg;
    a.eend = eend;
    a.stop_work = stop_work;
    const int64_t tiles = std::max<int64_t>(1, (eend - ebeg + 7) / 8);
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>((tiles + S::W - 1) / S::W, (int64_t)c->grid_grad - spare));
    if (mode == 0) k_grad<N, MODE_AX><<<g, S::W * 32, c->smem_grad, s>>>(a);
    else k_grad<N, MODE_PCG_A><<<g, S::W * 32, c->smem_grad, s>>>(a);
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    return IPDG_OK;
  }

  static int ensure_w2(ipdg_ctx c) {
    if (c->W2) return IPDG_OK;
    CUDA_TRY(c, cudaMalloc(&c->W2, std::max<int64_t>(1, c->K + c->H) * 2 * T::NP * sizeof(double)));
    return IPDG_OK;
  }

  static int ax_split(ipdg_ctx c, const double* u, double* Au, double lambda, cudaStream_t s) {
    TRY(ensure_w2(c));
    SplitArgs a = sargs(c);
    a.W2 = c->W2;
    a.u = u;
    a.Au = Au;
    a.lambda = lambda;
    using S = TrS<N>;
    if (c->H > 0) {  // own rows, then halo rows (the same split as the overlapped PCG pass A)
      TRY(grad_launch(c, a, 0, 0, c->K, 1, s));
      TRY(grad_launch(c, a, 0, c->K, c->K + c->H, 0, s));
    } else {
      k_grad<N, MODE_AX><<<c->grid_grad, S::W * 32, c->smem_grad, s>>>(a);
      c->launches++;
    }
    if (lambda != 0.0) k_flux<N, MODE_AX, true><<<c->grid_flux[0][1], S::W * 32, c->smem_flux[1], s>>>(a);
    else k_flux<N, MODE_AX, false><<<c->grid_flux[0][0], S::W * 32, c->smem_flux[0], s>>>(a);
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    return IPDG_OK;
  }

  static int pass_a_split(ipdg_ctx c, cudaStream_t s) {
    TRY(ensure_w2(c));
    SplitArgs a = sargs(c);
    a.W2 = c->W2;
    a.lambda = c->lambda;
    a.z = c->precond ? c->zb : c->r;
    a.p_even = c->pe;
    a.p_odd = c->po;
    a.x = c->x;
    a.Au = c->Ap;
    a.st = c->st;
    a.partials = c->partials;
    a.counter = c->counter;
    using S = TrS<N>;
    if (c->H > 0) {  // own rows overlap the halo exchange (comm stream); halo rows once it has landed
      TRY(grad_launch(c, a, 1, 0, c->K, 1, s, c->halo_ev_pending ? kCommSlots : 0));
      if (c->halo_ev_pending) CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_halo, 0));
      TRY(grad_launch(c, a, 1, c->K, c->K + c->H, 0, s));
    } else {
      k_grad<N, MODE_PCG_A><<<c->grid_grad, S::W * 32, c->smem_grad, s>>>(a);
      c->launches++;
    }
    if (c->lambda != 0.0) k_flux<N, MODE_PCG_A, true><<<c->grid_flux[1][1], S::W * 32, c->smem_flux[1], s>>>(a);
    else k_flux<N, MODE_PCG_A, false><<<c->grid_flux[1][0], S::W * 32, c->smem_flux[0], s>>>(a);
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    return IPDG_OK;
  }

  static AxArgs args(ipdg_ctx c) {
    AxArgs a;
    std::memset(&a, 0, sizeof(a));
    a.K = c->K;
    a.H = c->H;
    a.nblocks = c->nblocks;
    a.geo = c->geo;
    a.nbr = c->nbr;
    a.goff = c->goff;
    a.gid = c->gid;
    a.boff = c->boff;
    a.tables = c->tables;
    a.gG = c->gG;
    a.gF = c->gF;
    a.nbg = c->nbg;
    a.tau_c = c->tau_c;
    a.halo_p = c->halobuf;
    return a;
  }

  static int ax(ipdg_ctx c, const double* u, double* Au, double lambda, cudaStream_t s) {
    const bool lam = lambda != 0.0;
    const int k = resolve(c, 0, lam, u);
    if (k == 2) return ax_split(c, u, Au, lambda, s);
    AxArgs a = args(c);
    a.u = u;
    a.Au = Au;
    a.lambda = lambda;
    if (k == 5) return launch_gather<MODE_AX>(c, a, lam, s);
    if (k == 6) {
      if (!aligned16(Au)) FAIL(c, IPDG_EINVAL, "k_tpb: Au must be 16-byte aligned");
      return launch_tpb<MODE_AX>(c, a, lam, s, nullptr, 0);
    }
    if (k == 4) {
      const int gp = c->grid_pipe[0][lam];
      if (lam) k_pipe<N, MODE_AX, true><<<gp, T::W * 32, c->smem_pipe[0][1], s>>>(a, c->gmax);
      else k_pipe<N, MODE_AX, false><<<gp, T::W * 32, c->smem_pipe[0][0], s>>>(a, c->gmax);
      c->launches++;
      CUDA_TRY(c, cudaGetLastError());
      return IPDG_OK;
    }
    const int g = c->grid[0][lam];
    if (lam) k_sipdg<N, MODE_AX, true><<<g, T::W * 32, c->smem[0][1], s>>>(a, c->gmax);
    else k_sipdg<N, MODE_AX, false><<<g, T::W * 32, c->smem[0][0], s>>>(a, c->gmax);
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    return IPDG_OK;
  }

  static int pass_a(ipdg_ctx c, cudaStream_t s) {
    const int k = resolve(c, 1, c->lambda != 0.0, c->x);
    if (k == 2) return pass_a_split(c, s);
    AxArgs a = args(c);
    a.lambda = c->lambda;
    a.r = c->r;
    a.dinv = c->precond ? c->dinv : nullptr;
    a.z = c->precond ? c->zb : c->r;
    a.p_even = c->pe;
    a.p_odd = c->po;
    a.x = c->x;
    a.defer_x = c->xb ? 0 : 1;
    a.Au = c->Ap;
    a.st = c->st;
    a.partials = c->partials;
    a.counter = c->counter;
    const bool lam = c->lambda != 0.0;
    if (k == 5) return launch_gather<MODE_PCG_A>(c, a, lam, s);
    if (k == 6) {
      a.defer_x = c->xb ? 0 : 1;
      if (c->split_a) {  // interior blocks, (wait for the halo exchange), halo-boundary blocks
        const int ni = c->nbt_split[0], nbd = c->nbt_split[1];
        a.red_part = (ni > 0 && nbd > 0) ? 1 : 0;
        if (ni > 0) TRY(launch_tpb<MODE_PCG_A>(c, a, lam, s, c->blist_t, ni, c->halo_ev_pending));
        if (c->halo_ev_pending) CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_halo, 0));
        a.red_part = (ni > 0 && nbd > 0) ? 2 : 0;
        if (nbd > 0) TRY(launch_tpb<MODE_PCG_A>(c, a, lam, s, c->blist_t + ni, nbd));
        return IPDG_OK;
      }
      return launch_tpb<MODE_PCG_A>(c, a, lam, s, nullptr, 0);
    }
    if (k == 4) {
      const int gp = c->grid_pipe[1][lam];
      auto launch = [&](int part, const int* list, int n) -> int {
        a.blist = list;
        a.nlist = n;
        a.red_part = part;
        // while the exchange is in flight leave a few CTA slots free for NCCL's kernel (the persistent grid
        // would otherwise fill every SM and the exchange could only start after the interior blocks)
        const int cap = (part == 1 && c->halo_ev_pending) ? std::max(1, gp - kCommSlots) : gp;
        const int g = list ? std::max(1, std::min(cap, n)) : gp;
        if (lam) k_pipe<N, MODE_PCG_A, true><<<g, T::W * 32, c->smem_pipe[1][1], s>>>(a, c->gmax);
        else k_pipe<N, MODE_PCG_A, false><<<g, T::W * 32, c->smem_pipe[1][0], s>>>(a, c->gmax);
        c->launches++;
        CUDA_TRY(c, cudaGetLastError());
        return IPDG_OK;
      };
      if (c->split_a) {  // interior blocks, (wait for the halo exchange), halo-boundary blocks
        TRY(launch(1, c->blist, c->nb_split[0]));
        if (c->halo_ev_pending) CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_halo, 0));
        return launch(2, c->blist + c->nb_split[0], c->nb_split[1]);
      }
      return launch(0, nullptr, 0);
    }
    const int g = c->grid[1][lam];
    if (lam) k_sipdg<N, MODE_PCG_A, true><<<g, T::W * 32, c->smem[1][1], s>>>(a, c->gmax);
    else k_sipdg<N, MODE_PCG_A, false><<<g, T::W * 32, c->smem[1][0], s>>>(a, c->gmax);
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    return IPDG_OK;
  }

  // block-Jacobi (scaled inverse mass) residual pass: init (r = b - Ax0) or update (r -= alpha Ap)
  static int pass_b_bj(ipdg_ctx c, bool init, const double* b, cudaStream_t s) {
    constexpr int EPB = 256 / T::NP;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((c->K + EPB - 1) / EPB, (int64_t)c->sms * 8));
    if (init)
      k_pcg_bj<N, true><<<grid, 256, 0, s>>>(c->K, b, c->Ap, c->r, c->zb, c->gG, c->Minv, c->lambda, c->st, c->partials,
                                             c->counter, nullptr, nullptr, nullptr);
    else
      k_pcg_bj<N, false><<<grid, 256, 0, s>>>(c->K, c->r, c->Ap, c->r, c->zb, c->gG, c->Minv, c->lambda, c->st,
                                              c->partials, c->counter, c->xb ? c->x : nullptr, c->pe, c->po);
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    return IPDG_OK;
  }

  // DG gradient (div = false: o0, o1 = G p) or divergence (div = true: o0 = D u) with central fluxes
  static int dgop(ipdg_ctx c, bool div, const double* f0, const double* f1, double* o0, double* o1, cudaStream_t s) {
    if constexpr (N <= 4) {  // thread per element, operators in constant memory
      const int grid = (int)std::max<int64_t>(1, (c->K + 127) / 128);  // 128-thread CTAs (register-heavy)
      if (div) k_dgop_tpe<N, true><<<grid, 128, 0, s>>>(c->K, f0, f1, c->geo, c->nbg, o0, nullptr);
      else k_dgop_tpe<N, false><<<grid, 128, 0, s>>>(c->K, f0, nullptr, c->geo, c->nbg, o0, o1);
      c->launches++;
      CUDA_TRY(c, cudaGetLastError());
      return IPDG_OK;
    }
    constexpr int EPB = 256 / T::NP;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((c->K + EPB - 1) / EPB, (int64_t)c->sms * 8));
    if (div) {
      constexpr size_t bytes = dgop_smem_doubles<N, true>() * sizeof(double);
      CUDA_TRY(c, cudaFuncSetAttribute(k_dgop<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
      k_dgop<N, true><<<grid, 256, bytes, s>>>(c->K, f0, f1, c->geo, c->nbg, c->dgops, o0, nullptr);
    } else {
      constexpr size_t bytes = dgop_smem_doubles<N, false>() * sizeof(double);
      CUDA_TRY(c, cudaFuncSetAttribute(k_dgop<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
      k_dgop<N, false><<<grid, 256, bytes, s>>>(c->K, f0, nullptr, c->geo, c->nbg, c->dgops, o0, o1);
    }
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    return IPDG_OK;
  }

  // subcycling advection operator (NEXT-4, advect.cuh): fields = ub, vb, ut, vt; out = Nu, Nv
  static int advect(ipdg_ctx c, const double* const* fields, double* const* out, cudaStream_t s) {
    using A = TrA<N>;
    if (!c->adv_tab) {
      const AdvectOps ops = build_advect_ops(c->ref);
      if (ops.nc != A::NC || ops.ncf != A::NCF) FAIL(c, IPDG_ECUDA, "advection cubature size mismatch");
      // transposed layouts (coalesced across the threads of k_advect): IT [NP][NC], PrT / PsT [NC][NP]
      std::vector<double> t(A::NP * A::NC), pr(A::NC * A::NP), ps(A::NC * A::NP);
      for (int q = 0; q < A::NC; ++q)
        for (int j = 0; j < A::NP; ++j) {
          t[j * A::NC + q] = ops.I[q * A::NP + j];
          pr[q * A::NP + j] = ops.Pr[j * A::NC + q];
          ps[q * A::NP + j] = ops.Ps[j * A::NC + q];
        }
      t.insert(t.end(), pr.begin(), pr.end());
      t.insert(t.end(), ps.begin(), ps.end());
      t.insert(t.end(), ops.If.begin(), ops.If.end());
      t.insert(t.end(), ops.Lc.begin(), ops.Lc.end());
      TRY(upload(c, &c->adv_tab, t.data(), t.size()));
      const size_t bytes = (size_t)A::TOTAL * sizeof(double);
      CUDA_TRY(c, cudaFuncSetAttribute(k_advect<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    }
    AdvectArgs a;
    a.K = c->K;
    a.geo = c->geo;
    a.gG = c->gG;
    a.nbg = c->nbg;
    a.IT = c->adv_tab;
    a.PrT = a.IT + A::NC * A::NP;
    a.PsT = a.PrT + A::NP * A::NC;
    a.If = a.PsT + A::NP * A::NC;
    a.Lc = a.If + A::NCF * A::NFP;
    a.ub = fields[0];
    a.vb = fields[1];
    a.ut = fields[2];
    a.vt = fields[3];
    a.Nu = out[0];
    a.Nv = out[1];
    const int grid = (int)((c->K + A::EB - 1) / A::EB);
    k_advect<N><<<grid, A::NTHR, (size_t)A::TOTAL * sizeof(double), s>>>(a);
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    return IPDG_OK;
  }

  static int diag(ipdg_ctx c, double* d, double lambda, cudaStream_t s) {
    const int64_t n = c->K * T::NP;
    k_diag<N><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(c->K, c->geo, c->etoe, c->bcode, c->diagtab, c->tau_c, lambda, d);
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    return IPDG_OK;
  }

  static int mass(ipdg_ctx c, const double* u, double* Mu, cudaStream_t s) {
    const int64_t n = c->K * T::NP;
    k_mass<N><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(c->K, c->geo, c->Mref, u, Mu);
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    return IPDG_OK;
  }
};

#define IPDG_DEFINE_OPS(N_)                                                                                    \
  const ImplOps* impl_ops_##N_() {                                                                             \
    static const ImplOps ops = {Impl<N_>::build_tables, Impl<N_>::build_diagtab, Impl<N_>::configure,         \
                                Impl<N_>::resolve,      Impl<N_>::ax,            Impl<N_>::pass_a,            \
                                Impl<N_>::pass_b_bj,    Impl<N_>::dgop,          Impl<N_>::diag, Impl<N_>::mass,              \
                                Impl<N_>::upload_constants, Impl<N_>::advect}; \
    return &ops;                                                                                               \
  }
