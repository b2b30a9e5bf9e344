// Reference-triangle operators of degree N for libipdg (host C++17).
//
// Paper: arXiv:1801.00246 (P:n = PAPER.md line n).
//   P:56        Lagrange basis on Warp & Blend nodes (Warburton 2006), Np = (N+1)(N+2)/2
//   P:423-437   Eqs. elMass, elStiff, elLift: M, S = M D, LIFT = M^{-1} M^f
//   P:462-465   bi-unit reference triangle, read as {r,s >= -1, r+s <= 0} (R1)
// This is an independent implementation (it shares no code with oracle/): the 1-D
// Gauss-Lobatto points come from Newton iteration on P'_N instead of an
// eigen-solve, and all inverses use Gauss-Jordan elimination with partial pivoting.
#include "refops.h"

#include <cmath>
#include <stdexcept>

namespace ipdg {

namespace {

// Orthonormal Jacobi polynomial P_n^{(a,b)}(x) (weight (1-x)^a (1+x)^b on [-1,1]).
double jacobiP(double x, double a, double b, int n) {
  const double g0 = std::pow(2.0, a + b + 1) / (a + b + 1) * std::tgamma(a + 1) * std::tgamma(b + 1) /
                    std::tgamma(a + b + 1);
  double p0 = 1.0 / std::sqrt(g0);
  if (n == 0) return p0;
  const double g1 = (a + 1) * (b + 1) / (a + b + 3) * g0;
  double p1 = ((a + b + 2) * x / 2 + (a - b) / 2) / std::sqrt(g1);
  if (n == 1) return p1;
  double aold = 2 / (2 + a + b) * std::sqrt((a + 1) * (b + 1) / (a + b + 3));
  for (int i = 1; i < n; ++i) {
    const double h1 = 2 * i + a + b;
    const double anew =
        2 / (h1 + 2) * std::sqrt((i + 1) * (i + 1 + a + b) * (i + 1 + a) * (i + 1 + b) / (h1 + 1) / (h1 + 3));
    const double bnew = -(a * a - b * b) / h1 / (h1 + 2);
    const double p2 = (-aold * p0 + (x - bnew) * p1) / anew;
    aold = anew;
    p0 = p1;
    p1 = p2;
  }
  return p1;
}

double gradJacobiP(double x, double a, double b, int n) {
  if (n == 0) return 0.0;
  return std::sqrt(n * (n + a + b + 1)) * jacobiP(x, a + 1, b + 1, n - 1);
}

// Gauss-Lobatto points of degree N: -1, roots of P_{N-1}^{(1,1)}, +1 (Newton, Chebyshev start).
std::vector<double> gll_points(int N) {
  std::vector<double> x(N + 1);
  x[0] = -1.0;
  x[N] = 1.0;
  for (int k = 1; k < N; ++k) {
    double t = -std::cos(M_PI * k / N);
    for (int it = 0; it < 100; ++it) {
      const double f = jacobiP(t, 1, 1, N - 1);
      const double df = gradJacobiP(t, 1, 1, N - 1);
      const double dt = f / df;
      t -= dt;
      if (std::fabs(dt) < 1e-16) break;
    }
    x[k] = t;
  }
  return x;
}

// Gauss-Jordan inverse with partial pivoting (row-major n x n).
std::vector<double> invert(std::vector<double> A, int n) {
  std::vector<double> I(n * n, 0.0);
  for (int i = 0; i < n; ++i) I[i * n + i] = 1.0;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(A[r * n + c]) > std::fabs(A[piv * n + c])) piv = r;
    if (A[piv * n + c] == 0.0) throw std::runtime_error("singular matrix in reference-operator setup");
    if (piv != c)
      for (int j = 0; j < n; ++j) {
        std::swap(A[c * n + j], A[piv * n + j]);
        std::swap(I[c * n + j], I[piv * n + j]);
      }
    const double d = A[c * n + c];
    for (int j = 0; j < n; ++j) {
      A[c * n + j] /= d;
      I[c * n + j] /= d;
    }
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      const double f = A[r * n + c];
      if (f == 0.0) continue;
      for (int j = 0; j < n; ++j) {
        A[r * n + j] -= f * A[c * n + j];
        I[r * n + j] -= f * I[c * n + j];
      }
    }
  }
  return I;
}

std::vector<double> matmul(const std::vector<double>& A, const std::vector<double>& B, int n, int k, int m) {
  std::vector<double> C(n * m, 0.0);
  for (int i = 0; i < n; ++i)
    for (int l = 0; l < k; ++l) {
      const double a = A[i * k + l];
      for (int j = 0; j < m; ++j) C[i * m + j] += a * B[l * m + j];
    }
  return C;
}

std::vector<double> transpose(const std::vector<double>& A, int n, int m) {
  std::vector<double> T(m * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < m; ++j) T[j * n + i] = A[i * m + j];
  return T;
}

// 1-D warp function evaluated at x: interpolant (equidistant -> GLL displacement) / (1 - x^2).
double warp1d(int N, double x, const std::vector<double>& gll) {
  // Lagrange interpolation through the equidistant points of the displacement gll_i - eq_i
  double w = 0.0;
  for (int i = 0; i <= N; ++i) {
    const double xi = -1.0 + 2.0 * i / N;
    double li = 1.0;
    for (int j = 0; j <= N; ++j) {
      if (j == i) continue;
      const double xj = -1.0 + 2.0 * j / N;
      li *= (x - xj) / (xi - xj);
    }
    w += li * (gll[i] - xi);
  }
  if (std::fabs(x) < 1.0 - 1e-10) return w / (1.0 - x * x);
  return 0.0;  // the displacement vanishes at the end points
}

const double kAlphaOpt[15] = {0.0000, 0.0000, 1.4152, 0.1001, 0.2751, 0.9800, 1.0999, 1.2832,
                              1.3648, 1.4773, 1.4959, 1.5743, 1.5770, 1.6223, 1.6258};

void psi(int i, int j, double r, double s, double* v, double* dr, double* ds) {
  // orthonormal PKD mode sqrt(2) P_i(a) P_j^{(2i+1,0)}(b) (1-b)^i, a = 2(1+r)/(1-s) - 1, b = s
  const double a = (std::fabs(1.0 - s) > 1e-14) ? 2.0 * (1.0 + r) / (1.0 - s) - 1.0 : -1.0;
  const double b = s;
  const double fa = jacobiP(a, 0, 0, i), dfa = gradJacobiP(a, 0, 0, i);
  const double gb = jacobiP(b, 2 * i + 1, 0, j), dgb = gradJacobiP(b, 2 * i + 1, 0, j);
  const double hb = 0.5 * (1.0 - b);
  if (v) *v = std::sqrt(2.0) * fa * gb * std::pow(1.0 - b, i);
  // derivatives via d/dr = 2/(1-b) d/da ; d/ds = (1+a)/(1-b) d/da + d/db
  double dmr = dfa * gb * (i > 0 ? std::pow(hb, i - 1) : 1.0);
  double dms = dfa * gb * 0.5 * (1.0 + a) * (i > 0 ? std::pow(hb, i - 1) : 1.0);
  double t = dgb * std::pow(hb, i);
  if (i > 0) t -= 0.5 * i * gb * std::pow(hb, i - 1);
  dms += fa * t;
  const double sc = std::pow(2.0, i + 0.5);
  if (dr) *dr = dmr * sc;
  if (ds) *ds = dms * sc;
}

}  // namespace

RefOps build_refops(int N) {
  if (N < 1 || N > 8) throw std::invalid_argument("N out of range");
  RefOps R;
  R.N = N;
  R.Np = (N + 1) * (N + 2) / 2;
  R.Nfp = N + 1;
  const int Np = R.Np, Nfp = R.Nfp;
  const std::vector<double> gll = gll_points(N);
  R.gll = gll;
  // Warp & Blend nodes on the equilateral triangle, then barycentric map to (r,s)
  const double alpha = kAlphaOpt[N - 1];
  R.r.resize(Np);
  R.s.resize(Np);
  int sk = 0;
  for (int n = 0; n <= N; ++n) {
    for (int m = 0; m <= N - n; ++m) {
      const double L1 = double(n) / N, L3 = double(m) / N, L2 = 1.0 - L1 - L3;
      double x = -L2 + L3, y = (-L2 - L3 + 2.0 * L1) / std::sqrt(3.0);
      const double b1 = 4 * L2 * L3, b2 = 4 * L1 * L3, b3 = 4 * L1 * L2;
      const double w1 = b1 * warp1d(N, L3 - L2, gll) * (1 + (alpha * L1) * (alpha * L1));
      const double w2 = b2 * warp1d(N, L1 - L3, gll) * (1 + (alpha * L2) * (alpha * L2));
      const double w3 = b3 * warp1d(N, L2 - L1, gll) * (1 + (alpha * L3) * (alpha * L3));
      x += w1 + std::cos(2 * M_PI / 3) * w2 + std::cos(4 * M_PI / 3) * w3;
      y += std::sin(2 * M_PI / 3) * w2 + std::sin(4 * M_PI / 3) * w3;
      const double l1 = (std::sqrt(3.0) * y + 1.0) / 3.0;
      const double l2 = (-3.0 * x - std::sqrt(3.0) * y + 2.0) / 6.0;
      const double l3 = (3.0 * x - std::sqrt(3.0) * y + 2.0) / 6.0;
      R.r[sk] = -l2 + l3 - l1;
      R.s[sk] = -l2 - l3 + l1;
      ++sk;
    }
  }
  // Vandermonde V_{nk} = psi_k(r_n, s_n) and its gradients
  std::vector<double> V(Np * Np), Vr(Np * Np), Vs(Np * Np);
  for (int n = 0; n < Np; ++n) {
    int k = 0;
    for (int i = 0; i <= N; ++i)
      for (int j = 0; j <= N - i; ++j, ++k) psi(i, j, R.r[n], R.s[n], &V[n * Np + k], &Vr[n * Np + k], &Vs[n * Np + k]);
  }
  const std::vector<double> Vinv = invert(V, Np);
  R.Dr = matmul(Vr, Vinv, Np, Np, Np);
  R.Ds = matmul(Vs, Vinv, Np, Np, Np);
  R.M = matmul(transpose(Vinv, Np, Np), Vinv, Np, Np, Np);  // (V V^T)^{-1} = V^{-T} V^{-1}
  // Fmask: face 0 s=-1, face 1 r+s=0, face 2 r=-1 (ascending node index)
  R.Fmask.assign(3 * Nfp, -1);
  int c0 = 0, c1 = 0, c2 = 0;
  for (int n = 0; n < Np; ++n) {
    if (std::fabs(R.s[n] + 1) < 1e-10) R.Fmask[0 * Nfp + c0++] = n;
    if (std::fabs(R.r[n] + R.s[n]) < 1e-10) R.Fmask[1 * Nfp + c1++] = n;
    if (std::fabs(R.r[n] + 1) < 1e-10) R.Fmask[2 * Nfp + c2++] = n;
  }
  if (c0 != Nfp || c1 != Nfp || c2 != Nfp) throw std::runtime_error("Fmask construction failed");
  // 1-D face mass at the GLL points: (V1 V1^T)^{-1}, V1 from orthonormal Legendre
  std::vector<double> V1(Nfp * Nfp);
  for (int a = 0; a < Nfp; ++a)
    for (int k = 0; k < Nfp; ++k) V1[a * Nfp + k] = jacobiP(gll[a], 0, 0, k);
  const std::vector<double> V1inv = invert(V1, Nfp);
  R.M1D = matmul(transpose(V1inv, Nfp, Nfp), V1inv, Nfp, Nfp, Nfp);
  // E (Np x 3Nfp): face mass scattered to the face rows; LIFT = M^{-1} E = V V^T E
  std::vector<double> E(Np * 3 * Nfp, 0.0);
  for (int f = 0; f < 3; ++f)
    for (int a = 0; a < Nfp; ++a)
      for (int b = 0; b < Nfp; ++b) E[R.Fmask[f * Nfp + a] * 3 * Nfp + f * Nfp + b] = R.M1D[a * Nfp + b];
  const std::vector<double> VVt = matmul(V, transpose(V, Np, Np), Np, Np, Np);
  R.LIFT = matmul(VVt, E, Np, Np, 3 * Nfp);
  R.Minv = VVt;
  R.Sr = matmul(R.M, R.Dr, Np, Np, Np);
  R.Ss = matmul(R.M, R.Ds, Np, Np, Np);
  return R;
}

std::vector<double> interp_matrix(const RefOps& F, const RefOps& Cr) {
  const int nf = F.Np, nc = Cr.Np, N = Cr.N;
  std::vector<double> Vc(nc * nc), Vfc(nf * nc);
  for (int n = 0; n < nc; ++n) {
    int k = 0;
    for (int i = 0; i <= N; ++i)
      for (int j = 0; j <= N - i; ++j, ++k) psi(i, j, Cr.r[n], Cr.s[n], &Vc[n * nc + k], nullptr, nullptr);
  }
  for (int n = 0; n < nf; ++n) {
    int k = 0;
    for (int i = 0; i <= N; ++i)
      for (int j = 0; j <= N - i; ++j, ++k) psi(i, j, F.r[n], F.s[n], &Vfc[n * nc + k], nullptr, nullptr);
  }
  return matmul(Vfc, invert(Vc, nc), nf, nc, nc);
}

namespace {
// Gauss-Legendre rule on [-1, 1] (Newton on the three-term recurrence of P_n, Chebyshev start)
void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double t = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = t;
      for (int k = 1; k < n; ++k) {
        const double p2 = ((2 * k + 1) * t * p1 - k * p0) / (k + 1);
        p0 = p1;
        p1 = p2;
      }
      dp = n * (t * p1 - p0) / (t * t - 1.0);
      const double dt = p1 / dp;
      t -= dt;
      if (std::fabs(dt) < 1e-16) break;
    }
    x[n - 1 - i] = t;
    w[n - 1 - i] = 2.0 / ((1.0 - t * t) * dp * dp);
  }
}
}  // namespace

AdvectOps build_advect_ops(const RefOps& R) {
  const int N = R.N, Np = R.Np, Nfp = R.Nfp;
  const int n = (3 * N + 2) / 2 + 1;  // 2n - 1 >= 3N + 1 (the Duffy factor adds one degree in b)
  AdvectOps A;
  std::vector<double> g, gw;
  gauss_legendre(n, g, gw);
  A.nc = n * n;
  A.ncf = n;
  std::vector<double> rc(A.nc), sc(A.nc), wc(A.nc);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const double a = g[i], b = g[j];
      rc[i * n + j] = 0.5 * (1 + a) * (1 - b) - 1.0;
      sc[i * n + j] = b;
      wc[i * n + j] = gw[i] * gw[j] * 0.5 * (1 - b);
    }
  // Vandermonde of the nodes and of the cubature points (value and gradients)
  std::vector<double> V(Np * Np), Vc(A.nc * Np), Vcr(A.nc * Np), Vcs(A.nc * Np);
  for (int q = 0; q < Np; ++q) {
    int k = 0;
    for (int i = 0; i <= N; ++i)
      for (int j = 0; j <= N - i; ++j, ++k) psi(i, j, R.r[q], R.s[q], &V[q * Np + k], nullptr, nullptr);
  }
  for (int q = 0; q < A.nc; ++q) {
    int k = 0;
    for (int i = 0; i <= N; ++i)
      for (int j = 0; j <= N - i; ++j, ++k) psi(i, j, rc[q], sc[q], &Vc[q * Np + k], &Vcr[q * Np + k], &Vcs[q * Np + k]);
  }
  const std::vector<double> Vinv = invert(V, Np);
  A.I = matmul(Vc, Vinv, A.nc, Np, Np);                 // nc x Np
  const std::vector<double> Dcr = matmul(Vcr, Vinv, A.nc, Np, Np), Dcs = matmul(Vcs, Vinv, A.nc, Np, Np);
  const std::vector<double> Minv = R.Minv;             // M^{-1} = V V^T
  A.Pr.assign(Np * A.nc, 0.0);
  A.Ps.assign(Np * A.nc, 0.0);
  for (int nn = 0; nn < Np; ++nn)
    for (int q = 0; q < A.nc; ++q) {
      double pr = 0, ps = 0;
      for (int m = 0; m < Np; ++m) {
        pr += Minv[nn * Np + m] * Dcr[q * Np + m];
        ps += Minv[nn * Np + m] * Dcs[q * Np + m];
      }
      A.Pr[nn * A.nc + q] = pr * wc[q];
      A.Ps[nn * A.nc + q] = ps * wc[q];
    }
  // face points: Lagrange basis of the Nfp GLL face nodes (face parameter xi in face node order)
  std::vector<double> V1(Nfp * Nfp), V1g(n * Nfp);
  for (int a = 0; a < Nfp; ++a)
    for (int k = 0; k < Nfp; ++k) V1[a * Nfp + k] = jacobiP(R.gll[a], 0, 0, k);
  for (int a = 0; a < n; ++a)
    for (int k = 0; k < Nfp; ++k) V1g[a * Nfp + k] = jacobiP(g[a], 0, 0, k);
  A.If = matmul(V1g, invert(V1, Nfp), n, Nfp, Nfp);
  A.Lc.assign(Np * 3 * n, 0.0);
  for (int nn = 0; nn < Np; ++nn)
    for (int f = 0; f < 3; ++f)
      for (int j = 0; j < n; ++j) {
        double v = 0;
        for (int k = 0; k < Nfp; ++k) v += Minv[nn * Np + R.Fmask[f * Nfp + k]] * A.If[j * Nfp + k];
        A.Lc[nn * 3 * n + f * n + j] = v * gw[j];
      }
  return A;
}

}  // namespace ipdg
