// DG gradient and divergence with central fluxes: Eqs. INS_SD_4_1 / INS_SD_4_2,
// the operators on either side of the pressure solve -- its right-hand side -(gamma/dt) D.U and the
// velocity update U - (dt/gamma) G dP (Eq. INS_TD_3_3/3_4).  Nodal (strong) form per element:
//   G p = grad p + 1/2 sum_f (sJ/J) LIFT_f (n [[p]]),  D u = div u + 1/2 sum_f (sJ/J) LIFT_f (n.[[u]])
// with (sJ/J) n = g_f = -grad s, grad r + grad s, -grad r for faces 0, 1, 2, the jump [[w]] = w+ - w-
// (P:85), and homogeneous boundary mirrors read from the PRESSURE face codes (R20):
//   code 1 (pressure Dirichlet / outflow):  p+ = -p-, u+ = u-
//   code 2 (pressure Neumann / velocity Dirichlet): p+ = p-, u+ = -u-
// One thread per DOF of a chunk of 256 / Np elements; Dr, Ds, LIFT staged once per CTA in shared
// memory; the chunk's rows and the weighted face jumps go through shared memory.
#pragma once
#include "kernels.cuh"

namespace ipdg {

template <int N, bool DIV>
__global__ void __launch_bounds__(256) k_dgop(int64_t K, const double* __restrict__ f0, const double* __restrict__ f1,
                                              const double4* __restrict__ geo, const int4* __restrict__ nbg,
                                              const double* __restrict__ ops, double* __restrict__ o0,
                                              double* __restrict__ o1) {
  constexpr int NP = (N + 1) * (N + 2) / 2, NFP = N + 1, NF3 = 3 * NFP, EPB = 256 / NP, ACT = EPB * NP;
  extern __shared__ __align__(16) double sm[];
  double* Dr = sm;
  double* Ds = Dr + NP * NP;
  double* LIFT = Ds + NP * NP;           // [i][fk]
  double* r0 = LIFT + NP * NF3;          // chunk rows of f0
  double* r1 = r0 + ACT;                 // chunk rows of f1 (DIV)
  double* j0 = r1 + (DIV ? ACT : 0);     // G: g_x [[p]]; DIV: g.[[u]]     [el][fk]
  double* j1 = j0 + EPB * NF3;           // G: g_y [[p]]
  const int t = threadIdx.x;
  for (int q = t; q < 2 * NP * NP + NP * NF3; q += 256) sm[q] = ops[q];
  const int el = t / NP, i = t - el * NP;
  const bool active = t < ACT;
  for (int64_t e0 = (int64_t)blockIdx.x * EPB; e0 < K; e0 += (int64_t)gridDim.x * EPB) {
    const int64_t e = e0 + el;
    const bool ok = active && e < K;
    __syncthreads();  // previous chunk done with the shared rows
    if (ok) {
      r0[t] = f0[e * NP + i];
      if (DIV) r1[t] = f1[e * NP + i];
    }
    for (int q = t; q < EPB * NF3; q += 256) {  // weighted jumps at the face nodes of the chunk
      const int le = q / NF3, fk = q - le * NF3;
      const int64_t ee = e0 + le;
      if (ee >= K) continue;
      const int f = fk / NFP, k = fk - f * NFP;
      const int4 nb = nbg[ee];
      const int fl = (nb.w >> (4 * f)) & 15;
      const int fp = fl & 3, bc = fl >> 2;
      const double4 g = geo[ee];
      const double gx = (f == 0) ? -g.y : (f == 1) ? g.x + g.y : -g.x;
      const double gy = (f == 0) ? -g.w : (f == 1) ? g.z + g.w : -g.z;
      const int im = fmask_cf<N>(f, k);
      int64_t ip = ee * NP + im;
      double sgn = 1.0;
      if (bc == 0) {
        const int64_t n = (f == 0) ? nb.x : (f == 1) ? nb.y : nb.z;
        const int kp = ((f == 2) == (fp == 2)) ? NFP - 1 - k : k;
        ip = n * NP + fmask_cf<N>(fp, kp);
      } else {
        sgn = DIV ? (bc == 1 ? 1.0 : -1.0) : (bc == 1 ? -1.0 : 1.0);
      }
      const double a0 = f0[ee * NP + im];
      const double d0 = sgn * f0[ip] - a0;  // [[w]] = w+ - w-
      if (DIV) {
        const double a1 = f1[ee * NP + im];
        const double d1 = sgn * f1[ip] - a1;
        j0[q] = gx * d0 + gy * d1;
      } else {
        j0[q] = gx * d0;
        j1[q] = gy * d0;
      }
    }
    __syncthreads();
    if (ok) {
      const double4 g = geo[e];
      const double* row0 = r0 + el * NP;
      double dr0 = 0.0, ds0 = 0.0, dr1 = 0.0, ds1 = 0.0;
#pragma unroll 4
      for (int j = 0; j < NP; ++j) {
        dr0 = fma(Dr[i * NP + j], row0[j], dr0);
        ds0 = fma(Ds[i * NP + j], row0[j], ds0);
        if (DIV) {
          dr1 = fma(Dr[i * NP + j], r1[el * NP + j], dr1);
          ds1 = fma(Ds[i * NP + j], r1[el * NP + j], ds1);
        }
      }
      double l0 = 0.0, l1 = 0.0;
      const double* jr0 = j0 + el * NF3;
      const double* jr1 = j1 + el * NF3;
#pragma unroll 4
      for (int fk = 0; fk < NF3; ++fk) {
        l0 = fma(LIFT[i * NF3 + fk], jr0[fk], l0);
        if (!DIV) l1 = fma(LIFT[i * NF3 + fk], jr1[fk], l1);
      }
      if (DIV) {
        o0[e * NP + i] = g.x * dr0 + g.y * ds0 + g.z * dr1 + g.w * ds1 + 0.5 * l0;  // r_x, s_x, r_y, s_y
      } else {
        o0[e * NP + i] = g.x * dr0 + g.y * ds0 + 0.5 * l0;
        o1[e * NP + i] = g.z * dr0 + g.w * ds0 + 0.5 * l1;
      }
    }
  }
}

template <int N, bool DIV>
constexpr int dgop_smem_doubles() {
  constexpr int NP = (N + 1) * (N + 2) / 2, NF3 = 3 * (N + 1), EPB = 256 / NP, ACT = EPB * NP;
  return 2 * NP * NP + NP * NF3 + (DIV ? 2 : 1) * ACT + 2 * EPB * NF3;
}

}  // namespace ipdg

#include "cops.cuh"

namespace ipdg {

// Low-degree variant (N <= 4): one thread per element, operators as compile-time indices into
// __constant__ memory (c_tpe), the neighbour face values read from L1/L2 (as k_gather) -- no shared
// memory, no block barriers.  Same formulas as k_dgop.
template <int N, bool DIV>
__global__ void __launch_bounds__(128) k_dgop_tpe(int64_t K, const double* __restrict__ f0, const double* __restrict__ f1,
                                                  const double4* __restrict__ geo, const int4* __restrict__ nbg,
                                                  double* __restrict__ o0, double* __restrict__ o1) {
  using T = TrT<N>;
  constexpr int NP = T::NP, NFP = T::NFP, NF3 = T::NF3;
  const double* C = c_tpe<N>;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= K) return;
  double u0[NP], u1[NP];
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    u0[i] = f0[e * NP + i];
    u1[i] = DIV ? f1[e * NP + i] : 0.0;
  }
  const double4 g = geo[e];
  const int4 nb = nbg[e];
  double j0[NF3], j1[NF3];  // G: g_x [[p]], g_y [[p]];  DIV: g.[[u]] in j0
#pragma unroll
  for (int f = 0; f < 3; ++f) {
    const int fl = (nb.w >> (4 * f)) & 15;
    const int fp = fl & 3, bc = fl >> 2;
    const double gx = (f == 0) ? -g.y : (f == 1) ? g.x + g.y : -g.x;
    const double gy = (f == 0) ? -g.w : (f == 1) ? g.z + g.w : -g.z;
    const bool inner = (bc == 0);
    const int64_t n = (f == 0) ? nb.x : (f == 1) ? nb.y : nb.z;
    const bool flip = (f == 2) == (fp == 2);
    const double sgn = DIV ? (bc == 1 ? 1.0 : -1.0) : (bc == 1 ? -1.0 : 1.0);
#pragma unroll
    for (int k = 0; k < NFP; ++k) {
      const int im = fmask_cf<N>(f, k);
      double p0, p1 = 0.0;
      if (inner) {
        const int kp = flip ? NFP - 1 - k : k;
        const int ip = (fp == 0) ? fmask_cf<N>(0, kp) : (fp == 1) ? fmask_cf<N>(1, kp) : fmask_cf<N>(2, kp);
        p0 = f0[n * NP + ip];
        if (DIV) p1 = f1[n * NP + ip];
      } else {
        p0 = sgn * u0[im];
        if (DIV) p1 = sgn * u1[im];
      }
      const double d0 = p0 - u0[im];  // [[w]] = w+ - w-
      if (DIV) {
        j0[f * NFP + k] = gx * d0 + gy * (p1 - u1[im]);
      } else {
        j0[f * NFP + k] = gx * d0;
        j1[f * NFP + k] = gy * d0;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    double dr0 = 0.0, ds0 = 0.0, dr1 = 0.0, ds1 = 0.0, l0 = 0.0, l1 = 0.0;
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      dr0 = fma(C[T::O_DR + i * NP + j], u0[j], dr0);
      ds0 = fma(C[T::O_DS + i * NP + j], u0[j], ds0);
      if (DIV) {
        dr1 = fma(C[T::O_DR + i * NP + j], u1[j], dr1);
        ds1 = fma(C[T::O_DS + i * NP + j], u1[j], ds1);
      }
    }
#pragma unroll
    for (int fk = 0; fk < NF3; ++fk) {
      l0 = fma(C[T::O_LIFT + i * NF3 + fk], j0[fk], l0);
      if (!DIV) l1 = fma(C[T::O_LIFT + i * NF3 + fk], j1[fk], l1);
    }
    if (DIV) {
      o0[e * NP + i] = g.x * dr0 + g.y * ds0 + g.z * dr1 + g.w * ds1 + 0.5 * l0;
    } else {
      o0[e * NP + i] = g.x * dr0 + g.y * ds0 + 0.5 * l0;
      o1[e * NP + i] = g.z * dr0 + g.w * ds0 + 0.5 * l1;
    }
  }
}

}  // namespace ipdg
