"""Textbook (P)CG, the manufactured right-hand side and the L2 error (oracle; test infrastructure only).

P:219 -- the IP discretisation is symmetric positive-definite with the chosen
penalty, so the elliptic systems are solved by preconditioned conjugate
gradients.  P:221 / BASELINE config C4 -- point-Jacobi preconditioner
D = diag(A) (reading R11); P:221 -- for the screened Poisson operator
-L + lambda (lambda = gamma/(nu dt), Eq. ellipticOp1) the scaled inverse mass
matrix on each element (block-Jacobi).  The paper prints no tolerance, norm,
start or iteration cap (reading R12): stop when
||r_k||_2 <= tol ||b||_2 on the unpreconditioned residual, x0 given (0 in the
tests), checked every iteration, maxit from the caller.  Breakdown when
p^T A p <= 0; maxit reached is non-fatal.
Dot products are plain sequential sums (math.fsum is NOT used: numpy dot).
"""
import numpy as np

from . import meshops
from .quadrature import triangle_rule

OK, NOT_CONVERGED, BREAKDOWN = 0, 1, -4


def pcg(apply_A, b, tol, maxit, dinv=None, x0=None, apply_P=None):
    """Returns x, dict(iterations, rel_residual, status, history).

    Preconditioner: z = dinv * r (point Jacobi), z = apply_P(r) (any SPD block operator), or z = r."""
    if apply_P is None:
        apply_P = (lambda v: v * dinv) if dinv is not None else (lambda v: v.copy())
    b = np.asarray(b, dtype=np.float64).ravel()
    x = np.zeros_like(b) if x0 is None else np.asarray(x0, dtype=np.float64).ravel().copy()
    bnorm = np.sqrt(np.dot(b, b))
    if bnorm == 0.0:
        return np.zeros_like(b), dict(iterations=0, rel_residual=0.0, status=OK, history=[])
    r = b - apply_A(x) if np.any(x) else b.copy()
    z = apply_P(r)
    p = z.copy()
    rho = np.dot(r, z)
    rn = np.sqrt(np.dot(r, r))
    hist = [rn / bnorm]
    if rn <= tol * bnorm:
        return x, dict(iterations=0, rel_residual=rn / bnorm, status=OK, history=hist)
    for k in range(1, maxit + 1):
        q = apply_A(p)
        sigma = np.dot(p, q)
        if sigma <= 0.0:
            return x, dict(iterations=k, rel_residual=rn / bnorm, status=BREAKDOWN, history=hist)
        alpha = rho / sigma
        x = x + alpha * p
        r = r - alpha * q
        rn = np.sqrt(np.dot(r, r))
        hist.append(rn / bnorm)
        if rn <= tol * bnorm:
            return x, dict(iterations=k, rel_residual=rn / bnorm, status=OK, history=hist)
        z = apply_P(r)
        rho_new = np.dot(r, z)
        beta = rho_new / rho
        p = z + beta * p
        rho = rho_new
    return x, dict(iterations=maxit, rel_residual=rn / bnorm, status=NOT_CONVERGED, history=hist)


def inverse_mass_preconditioner(VX, VY, EToV, ref, lam):
    """"the scaled inverse mass matrix on each element" for the screened Poisson operator
    A = -L + lambda: z_e = (lambda J^e M)^{-1} r_e, the inverse of A's mass part lambda M^e,
    M^e = J^e M (Eq. elementOps).  Returns a callable on flat vectors."""
    if not lam > 0:
        raise ValueError("block-Jacobi inverse mass needs lambda > 0")
    J = meshops.affine_geometry(VX, VY, EToV)["J"]
    M = ref.M

    def apply(r):
        R = np.asarray(r, dtype=np.float64).reshape(-1, ref.Np)
        Z = np.linalg.solve(M, R.T).T / (lam * J[:, None])
        return Z.ravel()
    return apply


def rhs_mass_interp(VX, VY, EToV, ref, f):
    """b = J^e M f_I per element (reading R13): f interpolated at the nodes."""
    x, y = meshops.physical_nodes(VX, VY, EToV, ref)
    geo = meshops.affine_geometry(VX, VY, EToV)
    return geo["J"][:, None] * (f(x, y) @ ref.M.T)


def l2_error(VX, VY, EToV, ref, uh, uexact):
    """sqrt(sum_E int_E (u_h - u)^2) with a triangle rule exact to degree 2N+2; also ||u||."""
    rq, sq, wq = triangle_rule(ref.N + 2)
    V = ref.eval_basis(rq, sq)
    geo = meshops.affine_geometry(VX, VY, EToV)
    v = EToV
    xq = 0.5 * (-np.outer(VX[v[:, 0]], rq + sq) + np.outer(VX[v[:, 1]], 1 + rq) + np.outer(VX[v[:, 2]], 1 + sq))
    yq = 0.5 * (-np.outer(VY[v[:, 0]], rq + sq) + np.outer(VY[v[:, 1]], 1 + rq) + np.outer(VY[v[:, 2]], 1 + sq))
    uq = np.asarray(uh).reshape(-1, ref.Np) @ V.T
    ue = uexact(xq, yq)
    err = np.sqrt(np.sum(geo["J"][:, None] * wq[None, :] * (uq - ue) ** 2))
    nrm = np.sqrt(np.sum(geo["J"][:, None] * wq[None, :] * ue ** 2))
    return err, nrm
