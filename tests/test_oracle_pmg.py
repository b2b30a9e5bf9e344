"""Pins of the p-multigrid oracle (oracle/pmg.py, R22-R26).

Each pin checks a piece against something other than the oracle's own formula: the coarsening schedule
against SPEC's worked example, interpolation against closed-form monomials, the restriction against an
explicitly assembled transpose, the Chebyshev step against the closed-form Chebyshev residual polynomial,
the power iteration against a dense eigen-solve, the cycle against the operator properties CG needs, and
the preconditioner against the direct solve and point Jacobi.
"""
import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

from oracle import pmg, solvers
from oracle.assemble import assemble
from oracle.refelem import RefElem
from paper_1801_00246_b200 import meshgen


def test_schedule_examples():
    # S:509 worked example "N=4 -> degrees (4,2,1)"; halving down to 1
    assert pmg.schedule(4) == [4, 2, 1]
    assert pmg.schedule(8) == [8, 4, 2, 1]
    assert pmg.schedule(6) == [6, 3, 1]
    assert pmg.schedule(5) == [5, 2, 1]
    assert pmg.schedule(1) == [1]


def _monomials(rng, deg, r, s):
    val = np.zeros_like(r)
    coef = {}
    for a in range(deg + 1):
        for b in range(deg + 1 - a):
            coef[(a, b)] = rng.standard_normal()
            val = val + coef[(a, b)] * r ** a * s ** b
    return coef, val


@pytest.mark.parametrize("N", range(2, 9))
def test_interpolation_exact_on_coarse_polynomials(N):
    fine, coarse = RefElem(N), RefElem(pmg.schedule(N)[1])
    I = pmg.interpolation(fine, coarse)
    rng = np.random.default_rng(N)
    for _ in range(3):
        coef, uc = _monomials(rng, coarse.N, coarse.r, coarse.s)
        uf = sum(c * fine.r ** a * fine.s ** b for (a, b), c in coef.items())
        assert np.abs(I @ uc - uf).max() <= 1e-12 * max(1.0, np.abs(uf).max())
    assert np.abs(I @ np.ones(coarse.Np) - 1.0).max() <= 1e-13  # constants stay constants


def test_restriction_is_the_transpose():
    fine, coarse = RefElem(4), RefElem(2)
    I = pmg.interpolation(fine, coarse)
    K = 7
    P = sp.kron(sp.identity(K), sp.csr_matrix(I)).tocsr()  # the global block-diagonal prolongation
    rng = np.random.default_rng(1)
    uc, vf = rng.standard_normal(K * coarse.Np), rng.standard_normal(K * fine.Np)
    assert np.allclose(pmg.prolong(I, uc), P @ uc, rtol=0, atol=1e-14)
    assert np.allclose(pmg.restrict(I, vf), P.T @ vf, rtol=0, atol=1e-14)
    assert abs(np.dot(pmg.prolong(I, uc), vf) - np.dot(uc, pmg.restrict(I, vf))) <= 1e-12


def _cheb_T(k, t):
    """Chebyshev polynomial of the first kind, closed form (cos / cosh)."""
    t = np.asarray(t, dtype=np.float64)
    out = np.empty_like(t)
    m = np.abs(t) <= 1
    out[m] = np.cos(k * np.arccos(t[m]))
    out[t > 1] = np.cosh(k * np.arccosh(t[t > 1]))
    out[t < -1] = (-1) ** k * np.cosh(k * np.arccosh(-t[t < -1]))
    return out


@pytest.mark.parametrize("steps,ratio", [(2, None), (5, 40.0), (16, 250.0)])
def test_chebyshev_matches_the_residual_polynomial(steps, ratio):
    """Zero start, D = I, A = diag(lam): the error after k steps is T_k((theta - lam)/delta) /
    T_k(theta/delta) times the initial error, so x = (1 - q(lam)) / lam * b (closed form); k = 2 on
    [lmax/10, 1.1 lmax] is the smoother (R24), k = 16 on [1.1 lmax/250, 1.1 lmax] the coarse level (R26)."""
    lam = np.linspace(0.002, 2.0, 60)
    A = sp.diags(lam).tocsr()
    b = np.random.default_rng(2).standard_normal(lam.size)
    lmax = 2.0
    c = 1.1 * lmax
    a = lmax / 10.0 if ratio is None else c / ratio
    theta, delta = 0.5 * (c + a), 0.5 * (c - a)
    q = _cheb_T(steps, (theta - lam) / delta) / _cheb_T(steps, np.array([theta / delta]))[0]
    x = pmg.chebyshev(A, np.ones_like(lam), b, lmax, steps=steps, a=None if ratio is None else a)
    assert np.abs(x - (1.0 - q) / lam * b).max() <= 1e-11 * np.abs(b / lam).max()
    # inside the interval the error is damped by at least 1/T_k(theta/delta)
    inside = (lam >= a) & (lam <= c)
    assert np.abs(q[inside]).max() <= 1.0 / _cheb_T(steps, np.array([theta / delta]))[0] + 1e-14


def _small(N, nx=5):
    m = meshgen.square(nx, jitter=0.2, diag="random", order="morton", seed=7,
                       tag=lambda x, y: np.where(y < 0.5, 1, 2).astype(np.int8))
    return m, pmg.PMG(m["VX"], m["VY"], m["EToV"], m["bc"], N)


@pytest.mark.parametrize("N", [2, 4])
def test_power_iteration_brackets_the_largest_eigenvalue(N):
    m, H = _small(N)
    for A, di, lm in zip(H.A, H.dinv, H.lmax):
        w = sla.eigh(A.toarray(), np.diag(1.0 / di), eigvals_only=True)  # D^{-1} A: A v = lam D v
        assert 0.9 * w.max() <= lm <= w.max() * (1 + 1e-12)


@pytest.mark.parametrize("N", [1, 3, 4])
def test_vcycle_is_a_fixed_spd_operator(N):
    m, H = _small(N)
    n = H.A[0].shape[0]
    rng = np.random.default_rng(N)
    r1, r2 = rng.standard_normal(n), rng.standard_normal(n)
    B1, B2 = H.apply(r1), H.apply(r2)
    assert np.abs(H.apply(2.0 * r1 - 3.0 * r2) - (2.0 * B1 - 3.0 * B2)).max() <= 1e-11 * np.abs(B1).max()
    assert abs(np.dot(r2, B1) - np.dot(r1, B2)) <= 1e-11 * abs(np.dot(r1, B1))  # symmetric
    for _ in range(20):
        r = rng.standard_normal(n)
        assert np.dot(r, H.apply(r)) > 0.0  # positive
    assert np.abs(H.apply(np.zeros(n))).max() == 0.0


@pytest.mark.parametrize("N", [3, 4])
def test_pmg_pcg_converges_and_beats_jacobi(N):
    """PCG with the V-cycle reaches the direct solution and needs at most a third of point Jacobi's
    iterations (S:715's bar for the hybrid preconditioner against the unpreconditioned solve, here
    against the stronger Jacobi-PCG)."""
    m, H = _small(N, nx=8)
    A = H.A[0]
    b = solvers.rhs_mass_interp(m["VX"], m["VY"], m["EToV"], H.refs[0], meshgen.sin_sin_forcing).ravel()
    x, st = solvers.pcg(lambda v: A @ v, b, 1e-10, 5000, apply_P=H.apply)
    _, sj = solvers.pcg(lambda v: A @ v, b, 1e-10, 5000, dinv=H.dinv[0])
    assert st["status"] == 0 and sj["status"] == 0
    assert st["iterations"] * 3 <= sj["iterations"], (st["iterations"], sj["iterations"])
    xd = sp.linalg.spsolve(A.tocsc(), b)
    assert np.linalg.norm(x - xd) <= 1e-8 * np.linalg.norm(xd)


def test_level_operators_are_the_rediscretised_sipdg_operators():
    m, H = _small(4)
    for d, A in zip(H.degrees, H.A):
        B = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], RefElem(d))
        assert abs(A - B).max() == 0.0


def test_iterations_grow_at_most_2x_under_refinement():
    """S:504 / S:715 (the paper's VortexPreconditioner trend): PCG + p-multigrid iteration counts grow by at
    most 2x across one uniform refinement at N = 3."""
    its = []
    for nx in (6, 12):
        m, H = _small(3, nx=nx)
        A = H.A[0]
        b = solvers.rhs_mass_interp(m["VX"], m["VY"], m["EToV"], H.refs[0], meshgen.sin_sin_forcing).ravel()
        _, st = solvers.pcg(lambda v: A @ v, b, 1e-8, 5000, apply_P=H.apply)
        its.append(st["iterations"])
    assert its[1] <= 2 * its[0], its
