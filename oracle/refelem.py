"""Reference triangle of degree N (oracle; test infrastructure only).

Follows PAPER.md:
  * P:56   -- Lagrange basis on Warp & Blend nodes (Warburton 2006), N_p = (N+1)(N+2)/2.
  * P:423-437 (Eqs. elMass, elStiff, elLift) -- mass M, stiffness, derivative
    D = M^{-1} S, lift L^f = M^{-1} M^f on the reference element.
  * bi-unit reference triangle; read as {r,s >= -1, r+s <= 0}
    (reading R1: the printed "r+s <= 1" contradicts "bi-unit").
  * N_f = 3 faces, N_fp = N+1 nodes per face.

Node set: Warp & Blend construction on the equilateral triangle with the
optimised blending parameters alpha_opt(N) of Warburton (2006) (DESIGN.md
reading R2), mapped to (r,s).  Node order: row by row in s, r increasing.
Face order / Fmask (fixes trace orientation, reading R3):
  face 0: s = -1   (vertex 0 -> vertex 1)
  face 1: r+s = 0  (vertex 1 -> vertex 2)
  face 2: r = -1   (vertex 0 -> vertex 2)
each listed in ascending node index.
"""
import math

import numpy as np

from .quadrature import grad_jacobi_p, jacobi_gl, jacobi_p

ALPHA_OPT = [0.0000, 0.0000, 1.4152, 0.1001, 0.2751, 0.9800, 1.0999, 1.2832,
             1.3648, 1.4773, 1.4959, 1.5743, 1.5770, 1.6223, 1.6258]
NODETOL = 1e-10


def n_p(N):
    return (N + 1) * (N + 2) // 2


def vandermonde_1d(N, r):
    r = np.asarray(r, dtype=np.float64)
    V = np.zeros((r.size, N + 1))
    for j in range(N + 1):
        V[:, j] = jacobi_p(r, 0, 0, j)
    return V


def _warpfactor(N, rout):
    """1-D warp: interpolant of (GLL - equidistant) evaluated at rout, divided by the blend."""
    LGLr = jacobi_gl(0, 0, N)
    req = np.linspace(-1, 1, N + 1)
    Veq = vandermonde_1d(N, req)
    Pmat = np.array([jacobi_p(rout, 0, 0, i) for i in range(N + 1)])
    Lmat = np.linalg.solve(Veq.T, Pmat)
    warp = Lmat.T @ (LGLr - req)
    zerof = (np.abs(rout) < 1.0 - 1e-10).astype(np.float64)
    sf = 1.0 - (zerof * rout) ** 2
    return warp / sf + warp * (zerof - 1)


def nodes_equilateral(N):
    """Warp & Blend nodes (x, y) on the equilateral triangle (Warburton 2006)."""
    alpha = ALPHA_OPT[N - 1] if N < 16 else 5.0 / 3.0
    L1, L3 = [], []
    for n in range(1, N + 2):
        for m in range(1, N + 3 - n):
            L1.append((n - 1) / N)
            L3.append((m - 1) / N)
    L1 = np.array(L1)
    L3 = np.array(L3)
    L2 = 1.0 - L1 - L3
    x = -L2 + L3
    y = (-L2 - L3 + 2 * L1) / math.sqrt(3.0)
    blend1 = 4 * L2 * L3
    blend2 = 4 * L1 * L3
    blend3 = 4 * L1 * L2
    warpf1 = _warpfactor(N, L3 - L2)
    warpf2 = _warpfactor(N, L1 - L3)
    warpf3 = _warpfactor(N, L2 - L1)
    warp1 = blend1 * warpf1 * (1 + (alpha * L1) ** 2)
    warp2 = blend2 * warpf2 * (1 + (alpha * L2) ** 2)
    warp3 = blend3 * warpf3 * (1 + (alpha * L3) ** 2)
    x = x + warp1 + math.cos(2 * math.pi / 3) * warp2 + math.cos(4 * math.pi / 3) * warp3
    y = y + 0 * warp1 + math.sin(2 * math.pi / 3) * warp2 + math.sin(4 * math.pi / 3) * warp3
    return x, y


def xy_to_rs(x, y):
    """Equilateral (x,y) -> bi-unit (r,s) through barycentric coordinates."""
    L1 = (math.sqrt(3.0) * y + 1.0) / 3.0
    L2 = (-3.0 * x - math.sqrt(3.0) * y + 2.0) / 6.0
    L3 = (3.0 * x - math.sqrt(3.0) * y + 2.0) / 6.0
    return -L2 + L3 - L1, -L2 - L3 + L1


def rs_to_ab(r, s):
    """Collapsed coordinates a = 2(1+r)/(1-s) - 1, b = s (a = -1 at the top vertex)."""
    r = np.asarray(r, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    a = np.where(np.abs(1 - s) > 1e-14, 2 * (1 + r) / np.where(np.abs(1 - s) > 1e-14, 1 - s, 1.0) - 1, -1.0)
    return a, s


def simplex_basis(r, s, i, j):
    """Orthonormal PKD basis psi_ij = sqrt(2) P_i(a) P_j^{(2i+1,0)}(b) (1-b)^i."""
    a, b = rs_to_ab(r, s)
    return math.sqrt(2.0) * jacobi_p(a, 0, 0, i) * jacobi_p(b, 2 * i + 1, 0, j) * (1 - b) ** i


def grad_simplex_basis(r, s, i, j):
    """(d/dr, d/ds) of psi_ij, by the chain rule through (a, b)."""
    a, b = rs_to_ab(r, s)
    fa = jacobi_p(a, 0, 0, i)
    dfa = grad_jacobi_p(a, 0, 0, i)
    gb = jacobi_p(b, 2 * i + 1, 0, j)
    dgb = grad_jacobi_p(b, 2 * i + 1, 0, j)
    dmodr = dfa * gb
    if i > 0:
        dmodr = dmodr * (0.5 * (1 - b)) ** (i - 1)
    dmods = dfa * (gb * (0.5 * (1 + a)))
    if i > 0:
        dmods = dmods * (0.5 * (1 - b)) ** (i - 1)
    tmp = dgb * (0.5 * (1 - b)) ** i
    if i > 0:
        tmp = tmp - 0.5 * i * gb * (0.5 * (1 - b)) ** (i - 1)
    dmods = dmods + fa * tmp
    # psi carries sqrt(2) and (1-b)^i = 2^i (0.5(1-b))^i
    scale = 2.0 ** (i + 0.5)
    return dmodr * scale, dmods * scale


def basis_modes(N):
    return [(i, j) for i in range(N + 1) for j in range(N + 1 - i)]


def vandermonde_2d(N, r, s):
    return np.stack([simplex_basis(r, s, i, j) for (i, j) in basis_modes(N)], axis=1)


def grad_vandermonde_2d(N, r, s):
    cols = [grad_simplex_basis(r, s, i, j) for (i, j) in basis_modes(N)]
    return np.stack([c[0] for c in cols], axis=1), np.stack([c[1] for c in cols], axis=1)


class RefElem:
    """All reference-element data of degree N."""

    def __init__(self, N):
        if not 1 <= N <= 10:
            raise ValueError("degree N must satisfy 1 <= N <= 10")
        self.N = N
        self.Np = n_p(N)
        self.Nfp = N + 1
        x, y = nodes_equilateral(N)
        self.r, self.s = xy_to_rs(x, y)
        self.V = vandermonde_2d(N, self.r, self.s)
        self.Vinv = np.linalg.inv(self.V)
        Vr, Vs = grad_vandermonde_2d(N, self.r, self.s)
        # D = V_r V^{-1}: nodal derivative (Eq. elLift D = M^{-1} S on the reference element)
        self.Dr = Vr @ self.Vinv
        self.Ds = Vs @ self.Vinv
        # Eq. elMass on the reference element: M = (V V^T)^{-1}
        self.M = np.linalg.inv(self.V @ self.V.T)
        fm0 = np.nonzero(np.abs(self.s + 1) < NODETOL)[0]
        fm1 = np.nonzero(np.abs(self.r + self.s) < NODETOL)[0]
        fm2 = np.nonzero(np.abs(self.r + 1) < NODETOL)[0]
        self.Fmask = np.stack([fm0, fm1, fm2])  # 3 x Nfp
        # 1-D face mass at the face nodes (parameter in [-1,1] along the face)
        t0 = self.r[fm0]
        V1 = vandermonde_1d(N, t0)
        self.M1D = np.linalg.inv(V1 @ V1.T)
        # E (Np x 3Nfp): face mass M^f scattered to the face-node rows; LIFT = M^{-1} E (Eq. elLift)
        E = np.zeros((self.Np, 3 * self.Nfp))
        for f in range(3):
            E[np.ix_(self.Fmask[f], np.arange(f * self.Nfp, (f + 1) * self.Nfp))] = self.M1D
        self.E = E
        self.LIFT = self.V @ (self.V.T @ E)

    def lagrange_coeffs(self):
        """C with l_i(r,s) = sum_k C[i,k] psi_k(r,s)  (C = V^{-T})."""
        return self.Vinv.T

    def eval_basis(self, r, s):
        """Values (n x Np) of the nodal Lagrange basis at points (r,s)."""
        return vandermonde_2d(self.N, r, s) @ self.Vinv

    def eval_grad_basis(self, r, s):
        """(d/dr, d/ds) (each n x Np) of the nodal basis at points (r,s)."""
        Vr, Vs = grad_vandermonde_2d(self.N, r, s)
        return Vr @ self.Vinv, Vs @ self.Vinv
