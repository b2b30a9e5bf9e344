"""Pins for the oracle PCG (CPU only): SPEC worked examples, a direct solve, Jacobi."""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import solvers
from oracle.assemble import assemble
from oracle.refelem import RefElem
from paper_1801_00246_b200 import meshgen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_cg_2x2():
    g = GOLD["cg_2x2"]
    A = np.array(g["A"], dtype=float)
    x, st = solvers.pcg(lambda v: A @ v, np.array(g["b"], float), 1e-14, 10)
    assert np.allclose(x, g["x"], atol=1e-14) and st["status"] == solvers.OK and st["iterations"] <= 2


def test_cg_identity_one_iteration():
    b = np.random.default_rng(0).normal(size=50)
    x, st = solvers.pcg(lambda v: v, b, 1e-12, 10)
    assert st["iterations"] == GOLD["cg_identity"]["iterations"] and np.allclose(x, b)


def test_cg_zero_rhs_and_breakdown_and_maxit():
    x, st = solvers.pcg(lambda v: v, np.zeros(5), 1e-8, 10)
    assert st["iterations"] == 0 and not np.any(x)
    _, st = solvers.pcg(lambda v: -v, np.ones(3), 1e-8, 10)
    assert st["status"] == solvers.BREAKDOWN and st["iterations"] == 1
    A = np.diag(np.arange(1.0, 30.0))
    _, st = solvers.pcg(lambda v: A @ v, np.ones(29), 1e-14, 3)
    assert st["status"] == solvers.NOT_CONVERGED and st["iterations"] == 3


@pytest.mark.parametrize("precond", [False, True])
def test_pcg_matches_direct_solve_c1(precond):
    m = meshgen.square(4)
    ref = RefElem(2)
    A = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], ref)
    b = solvers.rhs_mass_interp(m["VX"], m["VY"], m["EToV"], ref, meshgen.sin_sin_forcing).ravel()
    dinv = 1.0 / A.diagonal() if precond else None
    x, st = solvers.pcg(lambda v: A @ v, b, 1e-12, 1000, dinv=dinv)
    xd = spla.spsolve(A.tocsc(), b)
    assert st["status"] == solvers.OK
    assert st["iterations"] <= A.shape[0]  # finite termination bound (exact arithmetic)
    r = b - A @ x
    assert np.linalg.norm(r) <= 1e-12 * np.linalg.norm(b) * (1 + 1e-6)
    kappa = np.linalg.cond(A.toarray())
    assert np.linalg.norm(x - xd) <= 10 * kappa * 1e-12 * np.linalg.norm(xd)
    # sqrt(kappa) iteration ceiling
    assert st["iterations"] <= int(np.ceil(0.5 * np.sqrt(kappa) * np.log(2 / 1e-12))) + 1


def test_jacobi_is_symmetric_and_helps():
    m = meshgen.square(12, jitter=0.2, diag="random", seed=1, tag=lambda x, y: np.where(x > 0.9, 1, 2))
    ref = RefElem(4)
    A = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], ref)
    b = np.random.default_rng(3).uniform(-1, 1, A.shape[0])
    _, s0 = solvers.pcg(lambda v: A @ v, b, 1e-8, 5000)
    _, s1 = solvers.pcg(lambda v: A @ v, b, 1e-8, 5000, dinv=1.0 / A.diagonal())
    assert s0["status"] == s1["status"] == solvers.OK
    assert s1["iterations"] < s0["iterations"]


@pytest.mark.parametrize("N", [1, 3, 5])
def test_inverse_mass_preconditioner_inverts_the_assembled_mass_part(N):
    """P:221 block-Jacobi: the preconditioner is the exact inverse of lambda * blockdiag(J^e M), checked
    against the quadrature assembly (A(lambda) - A(0) = lambda * mass), and it is symmetric."""
    m = meshgen.square(5, jitter=0.2, diag="random", order="morton", seed=4)
    ref = RefElem(N)
    lam = 7.0
    Ml = (assemble(m["VX"], m["VY"], m["EToV"], m["bc"], ref, lam=lam)
          - assemble(m["VX"], m["VY"], m["EToV"], m["bc"], ref, lam=0.0))
    P = solvers.inverse_mass_preconditioner(m["VX"], m["VY"], m["EToV"], ref, lam)
    rng = np.random.default_rng(5)
    v, w = rng.uniform(-1, 1, (2, Ml.shape[0]))
    assert np.linalg.norm(P(Ml @ v) - v) <= 1e-12 * np.linalg.norm(v)
    assert abs(w @ P(v) - v @ P(w)) <= 1e-12 * abs(w @ P(v))
    with pytest.raises(ValueError):
        solvers.inverse_mass_preconditioner(m["VX"], m["VY"], m["EToV"], ref, 0.0)


def test_block_jacobi_effective_for_mass_dominated_screened_poisson():
    """for small time steps the screened operator is dominated by the mass term, so the scaled
    inverse mass is an effective preconditioner (few iterations at large lambda = 1/(nu dt), fewer than
    point Jacobi), and its iteration count grows as the time step grows (smaller lambda); the solution
    matches a direct solve."""
    m = meshgen.square(6, jitter=0.2, diag="random", order="morton", seed=8)
    ref = RefElem(3)
    its = []
    for lam, cap in ((1e8, 4), (1e6, 8), (1e4, None), (1e2, None)):
        A = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], ref, lam=lam)
        b = np.random.default_rng(9).uniform(-1, 1, A.shape[0])
        P = solvers.inverse_mass_preconditioner(m["VX"], m["VY"], m["EToV"], ref, lam)
        x, st = solvers.pcg(lambda v: A @ v, b, 1e-10, 1000, apply_P=P)
        assert st["status"] == solvers.OK
        its.append(st["iterations"])
        if cap is not None:
            _, sj = solvers.pcg(lambda v: A @ v, b, 1e-10, 1000, dinv=1.0 / A.diagonal())
            assert st["iterations"] <= cap and st["iterations"] < sj["iterations"]
        xd = spla.spsolve(A.tocsc(), b)
        assert np.linalg.norm(x - xd) <= 1e-7 * np.linalg.norm(xd)
    assert its == sorted(its)
