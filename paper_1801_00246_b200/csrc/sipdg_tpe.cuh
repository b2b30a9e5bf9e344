// Thread-per-element variant of the SIPDG operator for low degree (N <= 4).
// Paper: arXiv:1801.00246; same formulation as kernels.cuh.  P:394 notes the "one thread to one
// element" mapping as the alternative to one thread per node.
//
// Every element's small dense products run as fully unrolled FP64 FMAs whose operator entries are
// compile-time indices into __constant__ memory, so each DFMA takes its operand from a uniform
// register (ULDC): no shared-memory traffic for operators, no padding, and the face structure is
// exploited (per-face LIFT^T S blocks, the face mass only on its N_fp rows) -- F close to F_min.
// Per element block (<= E own elements + <= GC ghost elements, one thread each):
//   P0  coalesced / TMA-free cp.async staging of the block's element rows into shared memory
//   A   all threads: u (PCG: p = z + beta p_{k-1}, deferred x update), [u_r, u_s] = [Dr u, Ds u],
//       w_r, w_s = J G (u_r, u_s) -> face traces t_f = sJ n.grad u at the face nodes -> smem
//   B   own threads: Au = Sr^T w_r + Ss^T w_s + sum_f [c_r,f (LIFT_f^T Sr)^T + c_s,f (LIFT_f^T Ss)^T] delta_f
//       - sum_f E_f (sJ g_f)  (+ lambda J M u), staged in smem and stored coalesced.
#pragma once
#include "kernels.cuh"

namespace ipdg {

template <int N_>
struct TrT {
  static constexpr int N = N_;
  static constexpr int NP = (N + 1) * (N + 2) / 2, NFP = N + 1, NF3 = 3 * NFP;
  static constexpr int E = 128;       // own elements per block
  static constexpr int GC = 64;       // ghost capacity per block
  static constexpr int NTHR = E + GC; // one thread per element slot
  // shared-memory row strides padded to an odd number of doubles: a warp reading one row per thread
  // then touches every bank pair once (conflict-free)
  static constexpr int NPS = NP | 1, NF3S = NF3 | 1;
  static constexpr int MINB = 2;  // resident CTAs per SM (register cap)
  // __constant__ table layout (doubles)
  static constexpr int O_DR = 0, O_DS = NP * NP, O_SR = 2 * NP * NP, O_SS = 3 * NP * NP;
  static constexpr int O_LSR = 4 * NP * NP;             // [fk][n]: (LIFT^T Sr)[fk][n]
  static constexpr int O_LSS = O_LSR + NF3 * NP;
  static constexpr int O_M1D = O_LSS + NF3 * NP;       // [k][m]
  static constexpr int O_M = O_M1D + NFP * NFP;         // [n][j] reference mass (lambda term)
  static constexpr int O_LIFT = O_M + NP * NP;          // [n][fk] LIFT (DG gradient / divergence, dgops.cuh)
  static constexpr int TOTAL = O_LIFT + NP * NF3;
};

template <int N>
__constant__ double c_tpe[TrT<N>::TOTAL];

struct TpeArgs {
  int64_t K;
  int nblocks;
  const int* boff;
  const int* goff;
  const int* gid;
  const short4* nbr;     // block-local slots (own < E, ghosts E + g) per face + (f' | bc << 2) << 4f
  const double4* geo;
  double tau_c, lambda;
  const double* u;
  const double* halo;
  double* Au;
  const double* z;
  double* p_even;
  double* p_odd;
  double* x;
  PcgState* st;
  double* partials;
  unsigned int* counter;
};

template <int N, bool PCG>
struct TpeSmem {
  using T = TrT<N>;
  // The staged operand rows are double-buffered (the next block's rows stream in while this one
  // computes) unless that would cost a resident CTA (N = 4 PCG).
  // stg[NB]: operand rows (own 0..E-1, ghosts E..E+GC-1) | trace t [slot][NF3] | det [slot] |
  // out rows [E][NP]; PCG adds po[NB]: p_{k-1} rows [slot][NP] | xs[NB]: x rows [E][NP]
  static constexpr int NB = (N <= 3 || !PCG) ? 2 : 1;
  static constexpr int SROWS = T::NTHR * T::NPS, XROWS = T::E * T::NPS;
  static constexpr int STG = 0;
  static constexpr int TRC = STG + NB * SROWS;
  static constexpr int DET = TRC + T::NTHR * T::NF3S;
  static constexpr int OUT = DET + T::NTHR;
  static constexpr int PO = OUT + T::E * T::NPS;
  static constexpr int GEO = PO + (PCG ? NB * SROWS : 0);  // [NB][slot] double4 geometry
  static constexpr int NBR = GEO + NB * T::NTHR * 4;         // [NB][own] short4 slots + face codes
  static constexpr int XS = NBR + NB * T::E;
  static constexpr int total() { return PCG ? XS + NB * XROWS : XS; }
};

template <int N, int MODE, bool LAM>
__global__ void __launch_bounds__(TrT<N>::NTHR, TrT<N>::MINB) k_tpe(TpeArgs a) {
  using T = TrT<N>;
  using L = TpeSmem<N, MODE == MODE_PCG_A>;
  constexpr int NP = T::NP, NFP = T::NFP, NF3 = T::NF3, E = T::E, NTHR = T::NTHR;
  constexpr int NPS = T::NPS, NF3S = T::NF3S;
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[32 * 3];
  double* stg = sm + L::STG;
  double* trc = sm + L::TRC;
  double* dets = sm + L::DET;
  double* outs = sm + L::OUT;
  double* pos = sm + L::PO;
  double* xs = sm + L::XS;
  const double* C = c_tpe<N>;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t K = a.K;
  PcgDecision d;
  double* pnew = nullptr;
  const double* pold = nullptr;
  const double* U = a.u;
  if (MODE == MODE_PCG_A) {
    PcgState* st = a.st;
    if (st->stop_iter >= 0) return;
    d = pcg_decide(st);
    pnew = (d.k & 1) ? a.p_odd : a.p_even;
    pold = (d.k & 1) ? a.p_even : a.p_odd;
    U = a.z;
    if (d.stop) {
      const int64_t n = K * NP;
      for (int64_t i = blockIdx.x * (int64_t)NTHR + tid; i < n; i += (int64_t)gridDim.x * NTHR) {
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
  double dot = 0.0;
  // ---- P0: stage a block's rows into buffer `buf` (own rows are one contiguous range)
  auto stage = [&](int b, int buf) {
    const int64_t e0 = a.boff[b];
    const int Eb = a.boff[b + 1] - a.boff[b];
    const int g0 = a.goff[b];
    const int Gb = a.goff[b + 1] - g0;
    double* sb = stg + buf * L::SROWS;
    double* pb = pos + buf * L::SROWS;
    double* xb = xs + buf * L::XROWS;
    double* gb = sm + L::GEO + buf * T::NTHR * 4;
    double* nbb = sm + L::NBR + buf * T::E;
    if (tid < Eb) {
      cp_async16(gb + tid * 4, &a.geo[e0 + tid].x);
      cp_async16(gb + tid * 4 + 2, &a.geo[e0 + tid].z);
      cp_async8(nbb + tid, &a.nbr[e0 + tid]);
    } else if (tid >= E && tid < E + Gb) {
      const int ge = a.gid[g0 + tid - E];
      cp_async16(gb + tid * 4, &a.geo[ge].x);
      cp_async16(gb + tid * 4 + 2, &a.geo[ge].z);
    }
    for (int q = tid; q < Eb * NP; q += NTHR) {
      const int o = (q / NP) * NPS + q % NP;
      cp_async8(sb + o, U + e0 * NP + q);
      if (MODE == MODE_PCG_A) {
        if (!d.first) cp_async8(pb + o, pold + e0 * NP + q);
        if (d.do_xupd) cp_async8(xb + o, a.x + e0 * NP + q);
      }
    }
    for (int q = tid; q < Gb * NP; q += NTHR) {
      const int g = q / NP, i = q - g * NP;
      const int ge = a.gid[g0 + g];
      const int o = (E + g) * NPS + i;
      if (ge >= K) {
        cp_async8(sb + o, a.halo + (int64_t)(ge - K) * NP + i);
      } else {
        cp_async8(sb + o, U + (int64_t)ge * NP + i);
        if (MODE == MODE_PCG_A && !d.first) cp_async8(pb + o, pold + (int64_t)ge * NP + i);
      }
    }
    cp_async_commit();
  };
  if (blockIdx.x < a.nblocks) stage(blockIdx.x, 0);
  int buf = 0;
  for (int b = blockIdx.x; b < a.nblocks; b += gridDim.x, buf = (L::NB == 2) ? buf ^ 1 : 0) {
    const int64_t e0 = a.boff[b];
    const int Eb = a.boff[b + 1] - a.boff[b];
    const int g0 = a.goff[b];
    const int Gb = a.goff[b + 1] - g0;
    if (L::NB == 2) {
      __syncthreads();  // the previous block is done with the other buffer
      if (b + (int)gridDim.x < a.nblocks) {
        stage(b + gridDim.x, buf ^ 1);
        cp_async_wait_group1();
      } else {
        cp_async_wait_all();
      }
    } else {
      if (b != (int)blockIdx.x) {
        __syncthreads();
        stage(b, 0);
      }
      cp_async_wait_all();
    }
    __syncthreads();
    double* stg = sm + L::STG + buf * L::SROWS;
    double* pos = sm + L::PO + buf * L::SROWS;
    double* xs = sm + L::XS + buf * L::XROWS;
    const double4* geos = reinterpret_cast<const double4*>(sm + L::GEO + buf * T::NTHR * 4);
    const short4* nbrs = reinterpret_cast<const short4*>(sm + L::NBR + buf * T::E);
    // ---- A: one thread per slot (own and ghost): gradient, w, face traces
    const bool own = tid < Eb;
    const bool ghost = tid >= E && tid < E + Gb;
    double wr[NP], ws[NP];
    if (own || ghost) {
      const int64_t el = own ? e0 + tid : (int64_t)a.gid[g0 + tid - E];
      double u[NP];
      double* row = stg + tid * NPS;
#pragma unroll
      for (int i = 0; i < NP; ++i) u[i] = row[i];
      if (MODE == MODE_PCG_A && !(ghost && el >= K)) {  // p_k = z + beta p_{k-1}
        const double* prow = pos + tid * NPS;
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          const double po = d.first ? 0.0 : prow[i];
          u[i] += d.beta * po;
          row[i] = u[i];  // p_k, stored coalesced with Au at the end of the block
        }
      }
      const double4 g = geos[tid];
      const double rx = g.x, sx = g.y, ry = g.z, sy = g.w;
      const double det = rx * sy - sx * ry;
      const double J = 1.0 / det;
      const double Grr = J * (rx * rx + ry * ry), Grs = J * (rx * sx + ry * sy), Gss = J * (sx * sx + sy * sy);
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
      // traces sJ n.grad u = -w_s, w_r + w_s, -w_r on faces 0, 1, 2
      double* tr = trc + tid * NF3S;
#pragma unroll
      for (int k = 0; k < NFP; ++k) {
        tr[k] = -ws[fmask_cf<N>(0, k)];
        tr[NFP + k] = wr[fmask_cf<N>(1, k)] + ws[fmask_cf<N>(1, k)];
        tr[2 * NFP + k] = -wr[fmask_cf<N>(2, k)];
      }
      dets[tid] = det;
    }
    __syncthreads();
    // ---- B: own threads: volume + lifted jumps + surface flux
    if (own) {
      const int64_t el = e0 + tid;
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
      const double4 g = geos[tid];
      const double rx = g.x, sx = g.y, ry = g.z, sy = g.w;
      const double det = dets[tid];
      const double J = 1.0 / det;
      const short4 nb = nbrs[tid];
      const double* uo = stg + tid * NPS;
      const double* to = trc + tid * NF3S;
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        const int fl = (nb.w >> (4 * f)) & 15;
        const int fp = fl & 3, bc = fl >> 2;
        const int slot = (f == 0) ? nb.x : (f == 1) ? nb.y : nb.z;
        const double gx = (f == 0) ? -sx : (f == 1) ? rx + sx : -rx;
        const double gy = (f == 0) ? -sy : (f == 1) ? ry + sy : -ry;
        const double sJ = J * sqrt(gx * gx + gy * gy);
        const bool inner = (bc == 0);
        const double detp = inner ? dets[slot] : 0.0;
        const double stau = sJ * a.tau_c * sJ * fmax(det, detp);  // sJ tau (Eq. Ch2.PenaltyParameter)
        const double cr = 0.5 * J * (rx * gx + ry * gy), cs = 0.5 * J * (sx * gx + sy * gy);
        const int ps = inner ? slot : tid;
        const int pf = inner ? fp : f;
        const bool flip = inner && ((f == 2) == (fp == 2));
        const double* un = stg + ps * NPS;
        const double* tn = trc + ps * NF3S + pf * NFP;
        double dr[NFP], ds[NFP], fg[NFP];
#pragma unroll
        for (int k = 0; k < NFP; ++k) {
          const int kp = flip ? NFP - 1 - k : k;
          const int ip = inner ? fmask_cf<N>(pf, kp) : fmask_cf<N>(f, k);
          const double um = uo[fmask_cf<N>(f, k)];
          const double tm = to[f * NFP + k];
          const double upr = un[ip], tp = tn[kp];
          const double delta = ((bc == 1) ? -upr : upr) - um;   // paper jump, mirrored on boundaries
          const double tq = (bc == 1) ? tp : -tp;              // sJ n-.grad u+
          dr[k] = cr * delta;
          ds[k] = cs * delta;
          fg[k] = -0.5 * (tm + tq) - stau * delta;             // -sJ (n.{grad u} + tau delta)
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
          for (int j = 0; j < NP; ++j) s = fma(C[T::O_M + n * NP + j], uo[j], s);
          out[n] = fma(lj, s, out[n]);
        }
      }
      double* orow = outs + tid * NPS;
#pragma unroll
      for (int n = 0; n < NP; ++n) {
        orow[n] = out[n];
        if (MODE == MODE_PCG_A) dot += uo[n] * out[n];
      }
    }
    __syncthreads();
    for (int q = tid; q < Eb * NP; q += NTHR) {  // coalesced stores
      const int o = (q / NP) * NPS + q % NP;
      a.Au[e0 * NP + q] = outs[o];
      if (MODE == MODE_PCG_A) {
        pnew[e0 * NP + q] = stg[o];
        if (d.do_xupd) a.x[e0 * NP + q] = fma(d.alpha_prev, pos[o], xs[o]);  // deferred x_{k-1} update
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
