// Subcycling advection operator N~(U_bar, U~): Eq. KSS_3,
// the volume part of Alg. SSV and the surface part of Alg. SSS, fused in one
// kernel; readings R27 (LLF sign of Alg. SSS) and R28 (velocity mirrors on boundaries).
//
//   N~ = -(r_x P_r F_x + s_x P_s F_x + r_y P_r F_y + s_y P_s F_y) + (1/J) sum_f sJ_f L_c^f (n.F~*)_f
//
// per advected component c in {u~, v~}: F = U_bar c at the volume cubature points (interpolated with I),
// n.F~* = 1/2 (n.U_bar- c- + n.U_bar+ c+) + 1/2 Lambda (c- - c+), Lambda = max |n.U_bar+-|, at the face
// cubature points (face values interpolated with If from the face nodes of both sides).  A CTA takes EB
// elements: their four rows are staged in shared memory; one thread per cubature point interpolates for
// all EB elements (each operator entry feeds 4 EB FMAs), one thread per (element, face point) forms the
// LLF flux, one thread per (node, group of EG elements) projects and lifts (8 EG FMAs per entry).  The
// operator tables (refops.cpp build_advect_ops, stored transposed) are read through the read-only cache.
#pragma once
#include "kernels.cuh"

namespace ipdg {

template <int N_>
struct TrA {
  static constexpr int N = N_;
  static constexpr int NP = (N + 1) * (N + 2) / 2, NFP = N + 1;
  static constexpr int NQ = (3 * N + 2) / 2 + 1;   // Gauss points per direction (exact to 3N)
  static constexpr int NC = NQ * NQ, NCF = NQ;      // volume points, points per face
  static constexpr int EB = N <= 5 ? 16 : 8;        // elements per CTA
  static constexpr int EG = 4;                      // elements per thread in the projection (register block)
  static constexpr int NTHR = 256;
  // shared memory (doubles): rows [NP][EB][4] | volume fluxes [4][EB][NC] | face fluxes [2][EB][3 NCF]
  static constexpr int S_U = 0, S_F = 4 * EB * NP, S_S = S_F + 4 * EB * NC, TOTAL = S_S + 2 * EB * 3 * NCF;
};

struct AdvectArgs {
  int64_t K;
  const double4* geo;  // r_x, s_x, r_y, s_y
  const double4* gG;   // .w = J
  const int4* nbg;     // neighbour per face (self on boundary) + flags (f' | bc << 2) << 4f
  const double *IT, *PrT, *PsT, *If, *Lc;  // IT [NP][NC], PrT / PsT [NC][NP] (transposed: coalesced)
  const double *ub, *vb, *ut, *vt;
  double *Nu, *Nv;
};

template <int N>
__global__ void __launch_bounds__(TrA<N>::NTHR) k_advect(AdvectArgs a) {
  using T = TrA<N>;
  constexpr int NP = T::NP, NFP = T::NFP, NC = T::NC, NCF = T::NCF, EB = T::EB, EG = T::EG, NTHR = T::NTHR;
  extern __shared__ __align__(16) double sm[];
  double* su = sm + T::S_U;  // [i][e][field], fields ub vb ut vt (one double4-like group per (i, e))
  double* sf = sm + T::S_F;  // [k][e][q], k: ub ut, vb ut, ub vt, vb vt
  double* ss = sm + T::S_S;  // [c][e][f NCF + j]: sJ (n.F~*)
  const int tid = threadIdx.x;
  const int64_t e0 = (int64_t)blockIdx.x * EB;
  const int Eb = (int)min((int64_t)EB, a.K - e0);
  const double* fld[4] = {a.ub, a.vb, a.ut, a.vt};
#pragma unroll
  for (int f = 0; f < 4; ++f)
    for (int q = tid; q < EB * NP; q += NTHR) {
      const int e = q / NP, i = q - e * NP;
      su[(i * EB + e) * 4 + f] = (e < Eb) ? fld[f][(e0 + e) * NP + i] : 0.0;
    }
  __syncthreads();
  // ---- volume cubature (Alg. SSV lines 3-9): one thread per point q for all EB elements -- every
  // interpolation entry I[q][j] is loaded once and feeds 4 EB FMAs
  for (int q = tid; q < NC; q += NTHR) {
    double acc[EB][4];
#pragma unroll
    for (int e = 0; e < EB; ++e)
#pragma unroll
      for (int f = 0; f < 4; ++f) acc[e][f] = 0.0;
    for (int j = 0; j < NP; ++j) {
      const double w = __ldg(a.IT + j * NC + q);
      const double4* uj = reinterpret_cast<const double4*>(su + j * EB * 4);
#pragma unroll
      for (int e = 0; e < EB; ++e) {
        const double4 u = uj[e];
        acc[e][0] = fma(w, u.x, acc[e][0]);
        acc[e][1] = fma(w, u.y, acc[e][1]);
        acc[e][2] = fma(w, u.z, acc[e][2]);
        acc[e][3] = fma(w, u.w, acc[e][3]);
      }
    }
#pragma unroll
    for (int e = 0; e < EB; ++e) {
      sf[(0 * EB + e) * NC + q] = acc[e][0] * acc[e][2];
      sf[(1 * EB + e) * NC + q] = acc[e][1] * acc[e][2];
      sf[(2 * EB + e) * NC + q] = acc[e][0] * acc[e][3];
      sf[(3 * EB + e) * NC + q] = acc[e][1] * acc[e][3];
    }
  }
  // ---- face cubature: LLF flux at the NCF points of each face (Alg. SSS lines 3-12, R27, R28)
  for (int t = tid; t < Eb * 3 * NCF; t += NTHR) {
    const int e = t / (3 * NCF), fj = t - e * 3 * NCF, f = fj / NCF, j = fj - f * NCF;
    const int64_t ge = e0 + e;
    const int4 nb = a.nbg[ge];
    const int fl = (nb.w >> (4 * f)) & 15, fp = fl & 3, bc = fl >> 2;
    const int64_t n = (f == 0) ? nb.x : (f == 1) ? nb.y : nb.z;
    const bool inner = (bc == 0);
    const bool flip = inner && ((f == 2) == (fp == 2));
    double m[4] = {0.0, 0.0, 0.0, 0.0}, p[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < NFP; ++k) {
      const double w = __ldg(a.If + j * NFP + k);
      const int im = fmask_cf<N>(f, k);
      const int kq = flip ? NFP - 1 - k : k;
      const int ip = fmask_cf<N>(fp, kq);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        m[c] = fma(w, su[(im * EB + e) * 4 + c], m[c]);
        if (inner) p[c] = fma(w, __ldg(fld[c] + n * NP + ip), p[c]);
      }
    }
    if (!inner) {  // R28 (R20 velocity types): outflow U+ = U-, velocity Dirichlet U+ = -U-
      const double sg = (bc == 2) ? -1.0 : 1.0;
#pragma unroll
      for (int c = 0; c < 4; ++c) p[c] = sg * m[c];
    }
    const double4 g = a.geo[ge];
    const double J = a.gG[ge].w;
    const double gx = (f == 0) ? -g.y : (f == 1) ? g.x + g.y : -g.x;  // sJ n = J g_f (k_geofacs)
    const double gy = (f == 0) ? -g.w : (f == 1) ? g.z + g.w : -g.z;
    const double gn = sqrt(gx * gx + gy * gy);
    const double nx = gx / gn, ny = gy / gn, sJ = J * gn;
    const double nUm = nx * m[0] + ny * m[1], nUp = nx * p[0] + ny * p[1];
    const double lam = fmax(fabs(nUm), fabs(nUp));
    ss[(0 * EB + e) * 3 * NCF + fj] = sJ * (0.5 * (nUm * m[2] + nUp * p[2]) + 0.5 * lam * (m[2] - p[2]));
    ss[(1 * EB + e) * 3 * NCF + fj] = sJ * (0.5 * (nUm * m[3] + nUp * p[3]) + 0.5 * lam * (m[3] - p[3]));
  }
  __syncthreads();
  // ---- project (Alg. SSV lines 10-18, with Eq. KSS_3's minus sign) and lift (Alg. SSS lines 13-18):
  // one thread per (node, group of EG elements) -- every projection entry feeds 8 EG FMAs
  constexpr int NGRP = EB / EG;
  for (int t = tid; t < NP * NGRP; t += NTHR) {
    const int nn = t % NP, eg = t / NP;
    double acc[EG][8];
#pragma unroll
    for (int e = 0; e < EG; ++e)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[e][k] = 0.0;
    for (int q = 0; q < NC; ++q) {
      const double wr = __ldg(a.PrT + q * NP + nn), ws = __ldg(a.PsT + q * NP + nn);
#pragma unroll
      for (int e = 0; e < EG; ++e) {
        const int ee = eg * EG + e;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double fv = sf[(k * EB + ee) * NC + q];
          acc[e][2 * k] = fma(wr, fv, acc[e][2 * k]);
          acc[e][2 * k + 1] = fma(ws, fv, acc[e][2 * k + 1]);
        }
      }
    }
    double lu[EG], lv[EG];
#pragma unroll
    for (int e = 0; e < EG; ++e) lu[e] = lv[e] = 0.0;
    const double* lc = a.Lc + nn * 3 * NCF;
    for (int q = 0; q < 3 * NCF; ++q) {
      const double w = __ldg(lc + q);
#pragma unroll
      for (int e = 0; e < EG; ++e) {
        const int ee = eg * EG + e;
        lu[e] = fma(w, ss[(0 * EB + ee) * 3 * NCF + q], lu[e]);
        lv[e] = fma(w, ss[(1 * EB + ee) * 3 * NCF + q], lv[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < EG; ++e) {
      const int ee = eg * EG + e;
      if (ee >= Eb) continue;
      const int64_t ge = e0 + ee;
      const double4 g = a.geo[ge];
      const double J = a.gG[ge].w;
      // g = (r_x, s_x, r_y, s_y): F_x = (k 0, k 2) for (u~, v~), F_y = (k 1, k 3); acc = (r, s) pairs per k
      a.Nu[ge * NP + nn] = -(g.x * acc[e][0] + g.y * acc[e][1] + g.z * acc[e][2] + g.w * acc[e][3]) + lu[e] / J;
      a.Nv[ge * NP + nn] = -(g.x * acc[e][4] + g.y * acc[e][5] + g.z * acc[e][6] + g.w * acc[e][7]) + lv[e] / J;
    }
  }
}

}  // namespace ipdg
