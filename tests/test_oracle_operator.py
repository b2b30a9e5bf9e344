"""Pins for the oracle SIPDG operator (CPU only).

Four routes and the mathematics fix the operator:
  * exact rational assembly (N <= 2) vs the float quadrature assembly;
  * quadrature assembly vs the matrix-free primal face loop;
  * symmetry, SPD, constants in the all-Neumann null space, the lambda-only term;
  * polynomial consistency: for a continuous polynomial p of degree <= N the
    SIPDG action on an element without boundary faces is J M (-Lap p)_I
    (integration by parts with zero jumps, from Eq. ellipticOp2);
  * O(h^{N+1}) L2 convergence of the manufactured sin(pi x) sin(pi y) problem.
A dropped term, wrong sign, transposed operand or wrong penalty breaks at least one.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import meshops, solvers
from oracle.assemble import assemble
from oracle.exact import assemble_exact
from oracle.mfree import MFree
from oracle.refelem import RefElem
from paper_1801_00246_b200 import meshgen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def _mixed_tag(xm, ym):
    return np.where(xm < 0.5, 1, 2).astype(np.int8)


MESHES = {
    "c1": lambda: meshgen.square(4),
    "jitter": lambda: meshgen.square(7, jitter=0.2, diag="random", order="morton", seed=2),
    "mixed": lambda: meshgen.square(6, jitter=0.2, diag="random", order="random", seed=3, tag=_mixed_tag),
}


@pytest.mark.parametrize("N", [1, 2])
@pytest.mark.parametrize("name", ["c1", "mixed_dyadic"])
def test_exact_rational_matches_float(N, name):
    if name == "c1":
        m = meshgen.square(4)
    else:
        m = meshgen.square(4, diag="random", seed=9, tag=_mixed_tag)
    Ae = assemble_exact(m["VX"], m["VY"], m["EToV"], m["bc"], N, lam=Fraction(3, 2))
    Af = np.array([[float(v) for v in row] for row in Ae])
    A = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], RefElem(N), lam=1.5).toarray()
    assert np.abs(A - Af).max() <= 2e-15 * np.abs(Af).max()
    # exact symmetry of the rational matrix
    n = len(Ae)
    assert all(Ae[i][j] == Ae[j][i] for i in range(n) for j in range(i))


@pytest.mark.parametrize("N", range(1, 9))
@pytest.mark.parametrize("name", ["c1", "jitter", "mixed"])
def test_assembled_equals_matrix_free(N, name):
    m = MESHES[name]()
    ref = RefElem(N)
    for lam in (0.0, 1.0):
        A = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], ref, lam=lam)
        mf = MFree(m["VX"], m["VY"], m["EToV"], m["bc"], ref)
        u = np.random.default_rng(100 + N).uniform(-1, 1, A.shape[0])
        a, b = A @ u, mf.apply(u, lam).ravel()
        assert np.linalg.norm(a - b) <= 1e-13 * np.linalg.norm(a)


@pytest.mark.parametrize("N", [1, 3, 5])
def test_symmetric_positive_definite(N):
    m = MESHES["mixed"]()
    A = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], RefElem(N)).toarray()
    assert np.abs(A - A.T).max() <= 1e-13 * np.abs(A).max()
    np.linalg.cholesky(A)  # raises unless SPD
    assert np.linalg.eigvalsh(A).min() > 0


@pytest.mark.parametrize("N", [1, 2, 4])
def test_neumann_null_space_and_lambda(N):
    m = meshgen.square(5, jitter=0.2, diag="random", seed=4, bc_code=2)
    ref = RefElem(N)
    A0 = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], ref)
    one = np.ones(A0.shape[0])
    assert np.abs(A0 @ one).max() < 1e-11 * abs(A0).max()
    lam = 2.5
    A1 = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], ref, lam=lam)
    from oracle.assemble import mass_matrix
    Mg = mass_matrix(m["VX"], m["VY"], m["EToV"], ref)
    assert np.abs(A1 @ one - lam * (Mg @ one)).max() < 1e-11 * abs(A1).max()
    assert np.linalg.eigvalsh(A0.toarray()).min() > -1e-10


POLYS = [  # (p, -Laplace p, min degree)
    (lambda x, y: 1.0 + 0 * x, lambda x, y: 0 * x, 1),
    (lambda x, y: 2 * x - 3 * y, lambda x, y: 0 * x, 1),
    (lambda x, y: x * x - y * y, lambda x, y: 0 * x, 2),
    (lambda x, y: x * x + y * y, lambda x, y: -4 + 0 * x, 2),
    (lambda x, y: x * y + y * y, lambda x, y: -2 + 0 * x, 2),
    (lambda x, y: x ** 3 - 3 * x * y * y + x * x * y, lambda x, y: -2 * y, 3),
]


@pytest.mark.parametrize("N", [1, 2, 3, 5])
def test_polynomial_consistency(N):
    m = meshgen.square(6, jitter=0.2, diag="random", seed=8)
    ref = RefElem(N)
    A = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], ref)
    x, y = meshops.physical_nodes(m["VX"], m["VY"], m["EToV"], ref)
    geo = meshops.affine_geometry(m["VX"], m["VY"], m["EToV"])
    interior = np.all(m["bc"] == 0, axis=1)
    for p, mlap, deg in POLYS:
        if deg > N:
            continue
        Ap = (A @ p(x, y).ravel()).reshape(-1, ref.Np)
        expect = geo["J"][:, None] * (mlap(x, y) @ ref.M.T)
        err = np.abs(Ap[interior] - expect[interior]).max()
        assert err < 1e-9 * max(1.0, np.abs(Ap).max()), err


@pytest.mark.parametrize("N", [1, 2, 3, 4])
def test_convergence_rate(N):
    """O(h^{N+1}) L2 error for u = sin(pi x) sin(pi y) (BASELINE config C1)."""
    ref = RefElem(N)
    errs, hs = [], []
    for nx in (4, 8, 16, 32):
        m = meshgen.square(nx)
        A = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], ref)
        b = solvers.rhs_mass_interp(m["VX"], m["VY"], m["EToV"], ref, meshgen.sin_sin_forcing).ravel()
        u = spla.spsolve(A.tocsc(), b)
        e, nrm = solvers.l2_error(m["VX"], m["VY"], m["EToV"], ref, u, meshgen.sin_sin)
        errs.append(e / nrm)
        hs.append(1.0 / nx)
    slope = np.polyfit(np.log(hs[-3:]), np.log(errs[-3:]), 1)[0]
    assert slope >= N + GOLD["convergence"]["min_slope_minus_N"], (slope, errs)
