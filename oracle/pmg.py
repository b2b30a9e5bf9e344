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
  R26 coarse      the AMG tail is out of scope, so the degree-1 level is solved approximately by a
                  longer Chebyshev polynomial: 16 steps over [1.1 lmax / 250, 1.1 lmax] (a fixed linear
                  symmetric operator, positive on the spectrum); with N = 1 it is the whole cycle.
  R25 cycle       one V-cycle with zero initial guess: x = S_l b; x += P_l V_{l+1}(R_l (b - A_l x));
                  x += S_l (b - A_l x); at level L: x = C_L b (R26).  S_l (the zero-start smoother) is a
                  polynomial in D^{-1}A times D^{-1}: symmetric, so the cycle is a fixed symmetric linear
                  operator, as CG requires.

Every function is written out step by step in that order; the matrix-vector products use the oracle's
assembled matrices (oracle.assemble).
"""
import numpy as np

from .assemble import assemble
from .refelem import RefElem, vandermonde_2d


# R26: the degree-1 level (no AMG tail) gets a longer Chebyshev polynomial over a wider interval
COARSE_STEPS, COARSE_RATIO = 16, 250.0


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


def chebyshev(A, dinv, b, lmax, steps=2, a=None):
    """R24: `steps` steps of the Chebyshev iteration for D^{-1} A x = D^{-1} b from x = 0 on [a, c],
    c = 1.1 lmax, a = lmax/10 (smoother; R26: the coarse level passes its own a and steps).  Textbook
    three-term form: theta = (c+a)/2, delta = (c-a)/2, sigma = theta/delta, rho_0 = 1/sigma,
    d_0 = D^{-1} r_0 / theta, then for m >= 1: rho_m = 1/(2 sigma - rho_{m-1}),
    d_m = rho_m rho_{m-1} d_{m-1} + (2 rho_m/delta) D^{-1} r_m, with x_{m+1} = x_m + d_m, r_m = b - A x_m."""
    c = 1.1 * lmax
    a = lmax / 10.0 if a is None else a
    theta, delta = 0.5 * (c + a), 0.5 * (c - a)
    sigma = theta / delta
    rho = 1.0 / sigma
    d = dinv * b / theta          # zero start: r_0 = b
    x = d
    for _ in range(steps - 1):
        rho_new = 1.0 / (2.0 * sigma - rho)
        r = b - A @ x
        d = rho_new * rho * d + (2.0 * rho_new / delta) * (dinv * r)
        x = x + d
        rho = rho_new
    return x


class PMG:
    """The hierarchy of R22-R26 for one mesh and fine degree N (lambda: the screening coefficient of
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
        if l == len(self.degrees) - 1:  # R26: coarse level
            return chebyshev(A, di, b, lm, steps=COARSE_STEPS, a=1.1 * lm / COARSE_RATIO)
        x = chebyshev(A, di, b, lm)
        r = b - A @ x
        xc = self.vcycle(restrict(self.I[l], r), l + 1)
        x = x + prolong(self.I[l], xc)
        r = b - A @ x
        return x + chebyshev(A, di, r, lm)

    def apply(self, r):
        return self.vcycle(np.asarray(r, dtype=np.float64).ravel())
