// FP64 SIPDG operator, Jacobi diagonal and PCG vector kernels for sm_100a.
// Paper: arXiv:1801.00246 (P:n = PAPER.md line n).  Formulation in kernels.cuh.
//
// Kernel k_sipdg<N, MODE, LAM> (one persistent CTA per SM slot, W warps):
//   per element block of E = 8W own elements plus the block's G ghost elements
//   (face neighbours outside the block, listed at setup):
//   P0  load u (or, in PCG pass A, form p = D^{-1} r + beta p_old on the fly) for own
//       and ghost elements, geometric factors, neighbour slots              -> smem
//   P1  per 8-element tile: [u_r | u_s] = u [Dr^T | Ds^T] on DMMA; own tiles keep
//       w_r, w_s = J G (u_r, u_s) in registers (C fragment layout); every tile writes
//       its face-node normal derivatives n.grad u to smem                   (Alg. AxG)
//   P2  per own face node: jump delta = u+ - u- (mirrored on boundary faces), flux
//       g = 1/2 n.(grad u- + grad u+) + tau delta, lift coefficients   (Alg. AxKernel)
//   P3  per own tile: Au = -sum_f sJ_f scatter(M1D g_f) (accumulator init)
//       + [w_r | w_s | face block] x [Sr; Ss; LIFT^T Sr; LIFT^T Ss] on DMMA (+ lambda J u M),
//       stored element-major; PCG pass A also accumulates p . Ap.
#include "kernels.cuh"

namespace ipdg {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

enum { MODE_AX = 0, MODE_PCG_A = 1 };

// shared-memory layout (in doubles) shared by host and device
struct SmemLayout {
  int tabG, tabM, tabL, m1d, iaux, us, dnt, geo, fa, gs, nb, total;  // offsets in doubles
  __host__ __device__ static int r2(int x) { return (x + 1) & ~1; }
  template <int N>
  __host__ __device__ static SmemLayout make(int gmax, bool lam) {
    using T = Tr<N>;
    SmemLayout L;
    const int gm8 = (gmax + 7) / 8 * 8;
    const int slots = T::E + gm8;
    int o = 0;
    L.tabG = o; o += T::TAB_G;
    L.tabM = o; o += T::TAB_M;
    L.tabL = o; o += lam ? T::TAB_L : 0;
    L.m1d = o; o += T::NFP * T::NFP;
    L.iaux = o; o += r2(T::NF3 + 2 * T::NPN) / 2;  // ints: fmask[NF3], nodeface[2*NPN]
    L.us = o; o += slots * T::SU;
    L.dnt = o; o += slots * T::NF3;
    L.geo = o; o += slots * 5;
    L.fa = o; o += T::E * T::SF;
    L.gs = o; o += T::E * T::NF3;
    L.nb = o; o += T::E;  // short4 per element = 8 bytes
    L.total = o;
    return L;
  }
};

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
  // last CTA: fixed-order sum over partials (strided per thread, then block tree)
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
__global__ void __launch_bounds__(Tr<N>::W * 32, 1) k_sipdg(AxArgs a, int gmax) {
  using T = Tr<N>;
  constexpr int NP = T::NP, NFP = T::NFP, NF3 = T::NF3, NT = T::NT, SU = T::SU, SF = T::SF;
  constexpr int W = T::W, E = T::E, KCG = T::KCG, KCW = T::KCW, KCF = T::KCF, KCM = T::KCM;
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[32 * 3];
  const SmemLayout L = SmemLayout::make<N>(gmax, LAM);
  double* tabG = sm + L.tabG;
  double* tabM = sm + L.tabM;
  double* tabL = sm + L.tabL;
  double* m1d = sm + L.m1d;
  int* fmask = reinterpret_cast<int*>(sm + L.iaux);
  int* nodeface = fmask + NF3;
  double* us = sm + L.us;
  double* dnt = sm + L.dnt;
  double* geos = sm + L.geo;
  double* fa = sm + L.fa;
  double* gs = sm + L.gs;
  short4* nbs = reinterpret_cast<short4*>(sm + L.nb);
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
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
      for (int64_t i = blockIdx.x * (int64_t)nthr + tid; i < n; i += (int64_t)gridDim.x * nthr) {
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

  // ---- stage the operator tables and small index tables once per CTA
  {
    const double* src = a.tables;
    const int ntab = T::TAB_G + T::TAB_M + (LAM ? T::TAB_L : 0);
    for (int i = tid; i < ntab; i += nthr) sm[i] = src[i];
    const double* aux = a.tables + T::TAB_G + T::TAB_M + T::TAB_L;
    for (int i = tid; i < NFP * NFP; i += nthr) m1d[i] = aux[i];
    const int* iaux = reinterpret_cast<const int*>(aux + NFP * NFP);
    for (int i = tid; i < NF3 + 2 * T::NPN; i += nthr) fmask[i] = iaux[i];
    // zero the padding columns once: u[NP..SU), face block [2*NF3..SF)
    const int slots = E + (gmax + 7) / 8 * 8;
    for (int i = tid; i < slots * SU; i += nthr) us[i] = 0.0;
    for (int i = tid; i < E * SF; i += nthr) fa[i] = 0.0;
  }

  double wr[NT][2], ws[NT][2];
  for (int b = blockIdx.x; b < a.nblocks; b += gridDim.x) {
    const int64_t e0 = a.boff[b];
    const int Eb = a.boff[b + 1] - a.boff[b];
    const int gbeg = a.goff[b];
    const int Gb = a.goff[b + 1] - gbeg;
    __syncthreads();
    // ---- P0: element data into shared memory
    for (int idx = tid; idx < Eb * NP; idx += nthr) {
      const int e = idx / NP, i = idx - e * NP;
      const int64_t g = e0 * NP + idx;
      double v;
      if (MODE == MODE_AX) {
        v = __ldg(a.u + g);
      } else {
        const double rr = __ldg(a.r + g);
        const double z = a.dinv ? rr * __ldg(a.dinv + g) : rr;
        const double po = first ? 0.0 : pold[g];
        v = first ? z : z + beta * po;
        pnew[g] = v;
        if (do_xupd) a.x[g] += alpha_prev * po;
      }
      us[e * SU + i] = v;
    }
    for (int idx = tid; idx < Gb * NP; idx += nthr) {
      const int gq = idx / NP, i = idx - gq * NP;
      const int ge = a.gid[gbeg + gq];
      double v;
      if (ge >= K) {
        v = a.halo_p[(int64_t)(ge - K) * NP + i];
      } else {
        const int64_t g = (int64_t)ge * NP + i;
        if (MODE == MODE_AX) {
          v = __ldg(a.u + g);
        } else {
          const double rr = __ldg(a.r + g);
          const double z = a.dinv ? rr * __ldg(a.dinv + g) : rr;
          v = first ? z : z + beta * pold[g];  // p_{k-1} of a ghost (owner writes p_k elsewhere)
        }
      }
      us[(E + gq) * SU + i] = v;
    }
    for (int s = tid; s < Eb + Gb; s += nthr) {
      const int slot = s < Eb ? s : E + (s - Eb);
      const int64_t el = s < Eb ? e0 + s : (int64_t)a.gid[gbeg + s - Eb];
      const double4 gg = a.geo[el];
      double* gp = geos + slot * 5;
      gp[0] = gg.x; gp[1] = gg.y; gp[2] = gg.z; gp[3] = gg.w;
      gp[4] = 1.0 / (gg.x * gg.w - gg.y * gg.z);  // J = 1 / det(G)
    }
    for (int e = tid; e < Eb; e += nthr) nbs[e] = a.nbr[e0 + e];
    __syncthreads();

    // ---- P1: reference gradient on DMMA, face normal derivatives, w_r / w_s
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
      const double* gp = geos + srow * 5;
      const double rx = gp[0], sx = gp[1], ry = gp[2], sy = gp[3], J = gp[4];
      // outward normals (unnormalised g_f = J^{-1} sJ n_f): -grad s, grad r + grad s, -grad r
      const double g0x = -sx, g0y = -sy, g1x = rx + sx, g1y = ry + sy, g2x = -rx, g2y = -ry;
      const double i0 = rsqrt(g0x * g0x + g0y * g0y), i1 = rsqrt(g1x * g1x + g1y * g1y), i2 = rsqrt(g2x * g2x + g2y * g2y);
      const double Grr = rx * rx + ry * ry, Grs = rx * sx + ry * sy, Gss = sx * sx + sy * sy;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = 8 * nt + 2 * (lane & 3) + h;
          const double ur = acc[nt][h], usv = acc[NT + nt][h];
          if (own) {
            wr[nt][h] = J * (Grr * ur + Grs * usv);
            ws[nt][h] = J * (Grs * ur + Gss * usv);
          }
          if (i < NP) {
            const double ux = rx * ur + sx * usv, uy = ry * ur + sy * usv;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int nf = nodeface[2 * i + q];
              if (nf >= 0) {
                const int f = nf / NFP;
                const double dn = (f == 0) ? (g0x * ux + g0y * uy) * i0
                                 : (f == 1) ? (g1x * ux + g1y * uy) * i1
                                            : (g2x * ux + g2y * uy) * i2;
                dnt[srow * NF3 + nf] = dn;
              }
            }
          }
        }
      }
    }
    __syncthreads();

    // ---- P2: jumps, fluxes and lift coefficients at the own face nodes
    for (int idx = tid; idx < Eb * NF3; idx += nthr) {
      const int e = idx / NF3, fk = idx - e * NF3;
      const int f = fk / NFP, kk = fk - f * NFP;
      const short4 nb = nbs[e];
      const int flags = nb.w;
      const int fl = (flags >> (4 * f)) & 15;
      const int fp = fl & 3, bc = fl >> 2;
      const int slot = (f == 0) ? nb.x : (f == 1) ? nb.y : nb.z;
      const double* gp = geos + e * 5;
      const double rx = gp[0], sx = gp[1], ry = gp[2], sy = gp[3], J = gp[4];
      const double gx = (f == 0) ? -sx : (f == 1) ? rx + sx : -rx;
      const double gy = (f == 0) ? -sy : (f == 1) ? ry + sy : -ry;
      const double glen = sqrt(gx * gx + gy * gy);
      const double sJ = J * glen;  // half edge length (R6)
      const double um = us[e * SU + fmask[fk]];
      const double dnm = dnt[e * NF3 + fk];
      double up, dnp, invJp;
      if (bc == 0) {
        const bool flip = ((f == 2) == (fp == 2));
        const int kp = flip ? NFP - 1 - kk : kk;
        up = us[slot * SU + fmask[fp * NFP + kp]];
        dnp = -dnt[slot * NF3 + fp * NFP + kp];  // neighbour's outward derivative, re-signed to n-
        invJp = 1.0 / geos[slot * 5 + 4];
      } else if (bc == 1) {  // Dirichlet mirror
        up = -um; dnp = dnm; invJp = 0.0;
      } else {               // Neumann mirror
        up = um; dnp = -dnm; invJp = 0.0;
      }
      const double delta = up - um;  // paper jump
      const double tau = a.tau_c * sJ * fmax(1.0 / J, invJp);  // Eq. Ch2.PenaltyParameter, 1/h = sJ/J
      const double gflux = 0.5 * (dnm + dnp) + tau * delta;
      // 1/2 sJ (r_x n_x + r_y n_y) = 1/2 J (r_x g_x + r_y g_y)
      fa[e * SF + fk] = 0.5 * J * (rx * gx + ry * gy) * delta;
      fa[e * SF + NF3 + fk] = 0.5 * J * (sx * gx + sy * gy) * delta;
      gs[e * NF3 + fk] = -sJ * gflux;
    }
    __syncthreads();

    // ---- P3: own tile of this warp -> Au
    if (8 * warp < Eb) {
      const int e = 8 * warp + (lane >> 2);
      double C[NT][2];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = 8 * nt + 2 * (lane & 3) + h;
          double s = 0.0;
          if (i < NP) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int nf = nodeface[2 * i + q];
              if (nf >= 0) {
                const int f = nf / NFP, kk = nf - f * NFP;
                const double* g = gs + e * NF3 + f * NFP;
#pragma unroll
                for (int m = 0; m < NFP; ++m) s += m1d[kk * NFP + m] * g[m];
              }
            }
          }
          C[nt][h] = s;
        }
      }
      // w_r, w_s straight from registers (K rows permuted on the host to match the C layout)
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
      const double* frow = fa + e * SF + (lane & 3);
#pragma unroll
      for (int kc = 0; kc < KCF; ++kc) {
        const double av = frow[4 * kc];
        const double* bt = tabM + (KCW + kc) * NT * 32 + lane;
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(C[j][0], C[j][1], av, bt[j * 32]);
      }
      if (LAM) {
        const double lj = a.lambda * geos[e * 5 + 4];
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
        double* out = (MODE == MODE_AX) ? a.Au : a.Au;
        const int64_t base = (e0 + e) * NP;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int i = 8 * nt + 2 * (lane & 3) + h;
            if (i < NP) {
              out[base + i] = C[nt][h];
              if (MODE == MODE_PCG_A) dot += us[e * SU + i] * C[nt][h];
            }
          }
      }
    }
  }
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
__global__ void __launch_bounds__(256) k_pcg_b(int64_t n, double* __restrict__ r, const double* __restrict__ Ap,
                                               const double* __restrict__ dinv, PcgState* st, double* partials,
                                               unsigned int* counter) {
  __shared__ double red[32 * 3];
  if (st->stop_iter >= 0) return;
  const long long k = st->it + 1;
  const double sigma = st->red_A;
  const double rho = st->rho_hist[(k - 1) & 3];
  if (!(sigma > 0.0)) {  // breakdown: p^T A p <= 0 (or NaN)
    double v[2] = {0.0, 0.0}, out[2];
    if (grid_reduce<2>(v, red, partials, counter, out)) {
      st->stop_iter = k;
      st->status = -4;
      st->final_rr = st->red_B[1];
      st->it = k;
    }
    return;
  }
  const double alpha = rho / sigma;
  double rz = 0.0, rr = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double ri = r[i] - alpha * Ap[i];
    r[i] = ri;
    const double zi = dinv ? ri * dinv[i] : ri;
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
__global__ void __launch_bounds__(256) k_pcg_init(int64_t n, const double* __restrict__ b, const double* __restrict__ Ax,
                                                  double* __restrict__ r, const double* __restrict__ dinv, PcgState* st,
                                                  double* partials, unsigned int* counter) {
  __shared__ double red[32 * 3];
  double rz = 0.0, rr = 0.0, bb = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double bi = b[i];
    const double ri = bi - Ax[i];
    r[i] = ri;
    const double zi = dinv ? ri * dinv[i] : ri;
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
__global__ void __launch_bounds__(256) k_pcg_final_x(int64_t n, double* __restrict__ x, const double* p_even,
                                                     const double* p_odd, const PcgState* st) {
  if (st->stop_iter >= 0) return;
  const long long k = st->it;
  if (k < 1) return;
  const double* p = (k & 1) ? p_odd : p_even;
  const double alpha = st->rho_hist[(k - 1) & 3] / st->red_A;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] += alpha * p[i];
}
__global__ void k_pcg_final_state(PcgState* st) {
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

__global__ void k_nodes(int64_t K, int NP, const double* __restrict__ vxy, const double* __restrict__ rs,
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
__global__ void k_geometry(int64_t K, const double* __restrict__ vxy, double4* __restrict__ geo,
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
