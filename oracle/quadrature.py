"""Orthogonal polynomials and quadrature rules (oracle; test infrastructure only).

The paper uses a nodal basis on Warp & Blend nodes and states the
element and face inner products (Eqs. elMass/elStiff) without
fixing a quadrature.  The oracle integrates them exactly with Gauss rules:
  * line:     Gauss-Legendre with n points, exact for degree 2n-1;
  * triangle: collapsed (Duffy) Gauss-Legendre x Gauss-Jacobi(1,0) rule on the
              bi-unit triangle {r,s >= -1, r+s <= 0} (SURVEY reading #1).
"""
import math

import numpy as np


def jacobi_p(x, alpha, beta, n):
    """Orthonormal Jacobi polynomial P_n^{(alpha,beta)}(x), weight (1-x)^a (1+x)^b.

    Three-term recurrence for the L2-normalised family (the basis of the
    orthonormal PKD construction used for the nodal Vandermonde).
    """
    x = np.asarray(x, dtype=np.float64)
    a, b = float(alpha), float(beta)
    gamma0 = 2.0 ** (a + b + 1) / (a + b + 1) * math.gamma(a + 1) * math.gamma(b + 1) / math.gamma(a + b + 1)
    p0 = np.full_like(x, 1.0 / math.sqrt(gamma0))
    if n == 0:
        return p0
    gamma1 = (a + 1) * (b + 1) / (a + b + 3) * gamma0
    p1 = ((a + b + 2) * x / 2 + (a - b) / 2) / math.sqrt(gamma1)
    if n == 1:
        return p1
    aold = 2 / (2 + a + b) * math.sqrt((a + 1) * (b + 1) / (a + b + 3))
    pm2, pm1 = p0, p1
    for i in range(1, n):
        h1 = 2 * i + a + b
        anew = 2 / (h1 + 2) * math.sqrt((i + 1) * (i + 1 + a + b) * (i + 1 + a) * (i + 1 + b) / (h1 + 1) / (h1 + 3))
        bnew = -(a * a - b * b) / h1 / (h1 + 2)
        p = (-aold * pm2 + (x - bnew) * pm1) / anew
        aold = anew
        pm2, pm1 = pm1, p
    return pm1


def grad_jacobi_p(x, alpha, beta, n):
    """d/dx of the orthonormal Jacobi polynomial: sqrt(n(n+a+b+1)) P_{n-1}^{(a+1,b+1)}."""
    x = np.asarray(x, dtype=np.float64)
    if n == 0:
        return np.zeros_like(x)
    return math.sqrt(n * (n + alpha + beta + 1)) * jacobi_p(x, alpha + 1, beta + 1, n - 1)


def jacobi_gq(alpha, beta, n):
    """n-point Gauss-Jacobi nodes/weights (Golub-Welsch on the Jacobi matrix)."""
    a, b = float(alpha), float(beta)
    if n == 1:
        x = np.array([(b - a) / (a + b + 2)])
        w = np.array([2.0 ** (a + b + 1) * math.gamma(a + 1) * math.gamma(b + 1) / math.gamma(a + b + 2)])
        return x, w
    k = np.arange(n, dtype=np.float64)
    h1 = 2 * k + a + b
    diag = np.empty(n)
    for i in range(n):
        if h1[i] == 0.0:  # k = 0 with a + b = 0: the limit value
            diag[i] = (b - a) / (a + b + 2)
        else:
            diag[i] = (b * b - a * a) / (h1[i] * (h1[i] + 2))
    kk = np.arange(1, n, dtype=np.float64)
    h = 2 * kk + a + b
    off = 2 / (h) * np.sqrt(kk * (kk + a + b) * (kk + a) * (kk + b) / (h - 1) / (h + 1))
    T = np.diag(diag) + np.diag(off, 1) + np.diag(off, -1)
    x, V = np.linalg.eigh(T)
    mu0 = 2.0 ** (a + b + 1) * math.gamma(a + 1) * math.gamma(b + 1) / math.gamma(a + b + 2)
    w = mu0 * V[0, :] ** 2
    return x, w


def jacobi_gl(alpha, beta, n):
    """Gauss-Lobatto points of degree n (n+1 points): -1, interior GQ(a+1,b+1,n-2), +1."""
    if n == 1:
        return np.array([-1.0, 1.0])
    xi, _ = jacobi_gq(alpha + 1, beta + 1, n - 1)
    return np.concatenate([[-1.0], np.sort(xi), [1.0]])


def line_rule(npts):
    """Gauss-Legendre rule on [-1,1] with npts points (exact to degree 2*npts-1)."""
    return jacobi_gq(0.0, 0.0, npts)


def triangle_rule(npts):
    """Collapsed Gauss rule on the bi-unit triangle, exact to degree 2*npts-1.

    (r, s) = ((1+a)(1-b)/2 - 1, b); dr ds = (1-b)/2 da db.  Gauss-Legendre in a,
    Gauss-Jacobi(1,0) in b absorbs the (1-b) factor.  Returns r, s, w.
    """
    a, wa = jacobi_gq(0.0, 0.0, npts)
    b, wb = jacobi_gq(1.0, 0.0, npts)
    A, B = np.meshgrid(a, b, indexing="ij")
    WA, WB = np.meshgrid(wa, wb, indexing="ij")
    r = (1 + A) * (1 - B) / 2 - 1
    s = B
    w = WA * WB / 2
    return r.ravel(), s.ravel(), w.ravel()
