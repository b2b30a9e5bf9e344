"""Matrix-free p-multigrid preconditioner for the SIPDG Poisson PCG (oracle; test infrastructure only).

Follows PAPER.md P:223-225: "we manually coarsen from degree N to degree 1 ...
implement the finest levels of the multigrid cycle in a matrix-free way", with the smoothing of P:223
("smoothing is chosen to be a degree 2 Chebyshev iteration").  The AMG coarse solve of pMG-AMG is out of
scope: the degree-1 level is only smoothed.  Every choice the paper leaves open is a
DESIGN.md reading:

  R22 levels      degrees N = d_0 > d_1 > ... > d_L = 1, d_{l+1} = max(1, floor(d_l / 2));
                  the level operator A_l is the SIPDG operator of degree d_l on the same mesh
                  (rediscretised, tau with its own (d_l+1)(d_l+2)/2 factor), applied matrix-free.
  R23 transfers   prolongation P_l: nodal interpolation of the degree-d_{l+1} polynomial at the degree-d_l
                  nodes, element by element; restriction R_l = P_l^T.
  R24 smoother    degree-2 Chebyshev iteration on D_l^{-1} A_l (D_l = diag A_l) over [lmax/10, 1.1 lmax],
                  lmax from 20 power iterations x <- D^{-1} A x / ||.||  (ratio of norms) from the fixed
                  start vector v_i = ((7919 i) mod 1009) / 1009 - 1/2 (i = global DOF index).
                  The coarsest level (degree 1) applies the same smoother once (no AMG tail).
  R25 cycle       one V-cycle with zero initial guess: x = S_l b; x += P_l V_{l+1}(R_l (b - A_l x));
                  x += S_l (b - A_l x); at level L: x = S_L b.  S_l (the zero-start smoother) is a
                  polynomial in D^{-1}A times D^{-1}: symmetric, so the cycle is a fixed symmetric linear
                  operator, as CG requires.

Every function is written out step by step in that order; the matrix-vector products use the oracle's
assembled matrices (oracle.assemble).
"""
import numpy as np

from .assemble import assemble
from .refelem import RefElem, vandermonde_2d


def schedule(N):
    """R22: N, floor(N/2), ..., 1."""
    d = [N]
    while d[-1] > 1:
        d.append(max(1, d[-1] // 2))
    return d


def interpolation(fine, coarse):
    """R23: (Np_f x Np_c) values of the degree-c nodal basis at the degree-f nodes."""
    return vandermonde_2d(coarse.N, fine.r, fine.s) @ coarse.Vinv


def prolong(I, uc):
    """Element-wise P: (K x Np_c) -> (K x Np_f) (flattened vectors)."""
    K = uc.size // I.shape[1]
    return (uc.reshape(K, I.shape[1]) @ I.T).ravel()


def restrict(I, rf):
    """Element-wise R = P^T: (K x Np_f) -> (K x Np_c)."""
    K = rf.size // I.shape[0]
    return (rf.reshape(K, I.shape[0]) @ I).ravel()


def start_vector(n):
    """R24: the fixed power-iteration start vector."""
    i = np.arange(n, dtype=np.int64)
    return ((7919 * i) % 1009) / 1009.0 - 0.5


def power_lmax(A, dinv, iters=20):
    """R24: lmax of D^{-1} A by 20 power iterations (ratio of norms)."""
    v = start_vector(A.shape[0])
    lam = 0.0
    for _ in range(iters):
        w = dinv * (A @ v)
        nw, nv = np.sqrt(np.dot(w, w)), np.sqrt(np.dot(v, v))
        lam = nw / nv
        v = w / nw
    return lam


def chebyshev(A, dinv, b, lmax):
    """R24: two steps of the Chebyshev iteration for D^{-1} A x = D^{-1} b from x = 0 on [a, c] = [lmax/10, 1.1 lmax]
    (textbook three-term form: theta = (c+a)/2, delta = (c-a)/2, sigma = theta/delta,
    rho_0 = 1/sigma, d_0 = D^{-1} r_0 / theta, rho_1 = 1/(2 sigma - rho_0),
    d_1 = rho_1 rho_0 d_0 + (2 rho_1/delta) D^{-1} r_1)."""
    a, c = lmax / 10.0, 1.1 * lmax
    theta, delta = 0.5 * (c + a), 0.5 * (c - a)
    sigma = theta / delta
    rho0 = 1.0 / sigma
    d = dinv * b / theta          # zero start: r_0 = b
    x = d
    rho1 = 1.0 / (2.0 * sigma - rho0)
    r = b - A @ x
    d = rho1 * rho0 * d + (2.0 * rho1 / delta) * (dinv * r)
    return x + d


class PMG:
    """The hierarchy of R22-R25 for one mesh and fine degree N (lambda: the screening coefficient of
    A = -L + lambda, the same on every level)."""

    def __init__(self, VX, VY, EToV, bc, N, lam=0.0):
        self.degrees = schedule(N)
        self.refs = [RefElem(d) for d in self.degrees]
        self.A = [assemble(VX, VY, EToV, bc, ref, lam=lam) for ref in self.refs]
        self.dinv = [1.0 / A.diagonal() for A in self.A]
        self.lmax = [power_lmax(A, di) for A, di in zip(self.A, self.dinv)]
        self.I = [interpolation(self.refs[l], self.refs[l + 1]) for l in range(len(self.degrees) - 1)]

    def vcycle(self, b, l=0):
        """R25."""
        A, di, lm = self.A[l], self.dinv[l], self.lmax[l]
        x = chebyshev(A, di, b, lm)
        if l == len(self.degrees) - 1:
            return x
        r = b - A @ x
        xc = self.vcycle(restrict(self.I[l], r), l + 1)
        x = x + prolong(self.I[l], xc)
        r = b - A @ x
        return x + chebyshev(A, di, r, lm)

    def apply(self, r):
        return self.vcycle(np.asarray(r, dtype=np.float64).ravel())
