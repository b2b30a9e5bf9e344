"""Pins of the subcycling advection oracle (oracle/advect.py; P:199-209 Eq. INS_CUB_N, Alg. SSV/SSS;
SURVEY 8.6 row f4; R27, R28).

  * consistency: for continuous polynomial fields the DG operator is exactly the element-wise L2
    projection of div(U_bar c), computed here from exact polynomial derivatives (oracle.exact) and a
    different, higher quadrature rule -- no basis gradients, no faces;
  * conservation: the element integrals of N~ sum to the boundary fluxes (interior LLF fluxes cancel);
  * the LLF sign (reading R27): for a constant U_bar, sum_E (c, N~ c)_E equals exactly
    1/2 sum_interior Lambda [[c]]^2 + 1/2 sum_boundary (n.U_bar) c^2 (dissipative, >= the boundary term).
"""
from fractions import Fraction as Fr

import numpy as np
import pytest

from oracle import advect, meshops
from oracle.exact import padd, pdiff, pmul
from oracle.quadrature import triangle_rule
from oracle.refelem import RefElem
from paper_1801_00246_b200 import meshgen


def _mesh(nx=5, tag=1, seed=8):
    return meshgen.square(nx, jitter=0.2, diag="random", order="morton", seed=seed,
                          tag=(lambda x, y: np.full_like(x, tag, dtype=np.int8)) if tag else
                          (lambda x, y: np.where(y < 0.5, 1, 2).astype(np.int8)))


def _peval(p, x, y):
    return sum(float(c) * x ** a * y ** b for (a, b), c in p.items())


def _rand_poly(rng, deg):
    return {(a, b): Fr(int(rng.integers(-9, 10)), 7) for a in range(deg + 1) for b in range(deg + 1 - a)}


@pytest.mark.parametrize("N", [1, 2, 3, 4, 6])
def test_continuous_fields_give_the_projected_divergence(N):
    m = _mesh(tag=1)  # all outflow: U+ = U- on the boundary, no jumps anywhere
    VX, VY, EToV = m["VX"], m["VY"], m["EToV"]
    ref = RefElem(N)
    rng = np.random.default_rng(N)
    ubp, vbp = _rand_poly(rng, 1), _rand_poly(rng, 1)
    utp, vtp = _rand_poly(rng, N), _rand_poly(rng, max(N - 1, 0))
    x, y = meshops.physical_nodes(VX, VY, EToV, ref)
    ub, vb, ut, vt = (_peval(p, x, y) for p in (ubp, vbp, utp, vtp))
    Nu, Nv = advect.advection(VX, VY, EToV, m["bc"], ref, ub, vb, ut, vt)
    geo = meshops.affine_geometry(VX, VY, EToV)
    rq, sq, wq = triangle_rule(2 * N + 3)
    V = ref.eval_basis(rq, sq)
    Minv = np.linalg.inv(ref.M)
    for out, cp in ((Nu, utp), (Nv, vtp)):
        div = padd(pdiff(pmul(ubp, cp), 0), pdiff(pmul(vbp, cp), 1))
        xq = 0.5 * (-np.outer(VX[EToV[:, 0]], rq + sq) + np.outer(VX[EToV[:, 1]], 1 + rq) + np.outer(VX[EToV[:, 2]], 1 + sq))
        yq = 0.5 * (-np.outer(VY[EToV[:, 0]], rq + sq) + np.outer(VY[EToV[:, 1]], 1 + rq) + np.outer(VY[EToV[:, 2]], 1 + sq))
        proj = (_peval(div, xq, yq) * wq[None]) @ V @ Minv.T  # M^{-1} (l, div F) on the reference element
        assert np.abs(out - proj).max() <= 1e-11 * max(1.0, np.abs(proj).max()), N
    del geo


@pytest.mark.parametrize("N", [2, 4])
def test_conservation(N):
    m = _mesh(tag=0)  # mixed outflow / wall
    ref = RefElem(N)
    K, Np = m["EToV"].shape[0], ref.Np
    rng = np.random.default_rng(3)
    ub, vb, ut, vt = (rng.uniform(-1, 1, (K, Np)) for _ in range(4))
    Nu, Nv = advect.advection(m["VX"], m["VY"], m["EToV"], m["bc"], ref, ub, vb, ut, vt)
    J = meshops.affine_geometry(m["VX"], m["VY"], m["EToV"])["J"]
    diag = advect.face_flux_integrals(m["VX"], m["VY"], m["EToV"], m["bc"], ref, ub, vb, ut, vt)
    one = np.ones(Np)
    for c, out in enumerate((Nu, Nv)):
        total = np.sum(J[:, None] * (out @ ref.M) * one[None])  # sum_E (1, N~)_E
        assert abs(total - diag[c, 0]) <= 1e-12 * max(1.0, np.abs(out).max() * K)


@pytest.mark.parametrize("N", [1, 3, 5])
def test_llf_energy_identity(N):
    """Constant advective velocity on an all-outflow mesh: the discrete energy production equals the
    interior LLF dissipation plus the boundary outflow term, exactly (Alg. SSS sign, R27)."""
    m = _mesh(tag=1)
    ref = RefElem(N)
    K, Np = m["EToV"].shape[0], ref.Np
    rng = np.random.default_rng(11)
    ub, vb = np.full((K, Np), 0.7), np.full((K, Np), -0.4)
    ut, vt = rng.uniform(-1, 1, (K, Np)), rng.uniform(-1, 1, (K, Np))
    Nu, Nv = advect.advection(m["VX"], m["VY"], m["EToV"], m["bc"], ref, ub, vb, ut, vt)
    J = meshops.affine_geometry(m["VX"], m["VY"], m["EToV"])["J"]
    diag = advect.face_flux_integrals(m["VX"], m["VY"], m["EToV"], m["bc"], ref, ub, vb, ut, vt)
    for c, (out, fld) in enumerate(((Nu, ut), (Nv, vt))):
        energy = np.sum(J[:, None] * fld * (out @ ref.M))  # sum_E (c, N~ c)_E  (M symmetric)
        assert abs(energy - (diag[c, 1] + diag[c, 2])) <= 1e-11 * max(1.0, abs(energy))
        assert diag[c, 1] > 0.0  # the random field jumps: strictly dissipative inside


def test_constant_fields_are_steady():
    m = _mesh(tag=1)
    ref = RefElem(3)
    K, Np = m["EToV"].shape[0], ref.Np
    c = [np.full((K, Np), v) for v in (0.3, -1.2, 2.0, 0.5)]
    Nu, Nv = advect.advection(m["VX"], m["VY"], m["EToV"], m["bc"], ref, *c)
    # rounding only: the flux scale |U|^2 / h is ~10 here
    assert np.abs(Nu).max() <= 1e-11 and np.abs(Nv).max() <= 1e-11
