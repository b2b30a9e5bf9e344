"""Pins for the oracle DG gradient / divergence with central fluxes (Eqs. INS_SD_4_1,
INS_SD_4_2).  CPU only."""
import numpy as np
import pytest

from oracle import dgops
from oracle.meshops import physical_nodes
from oracle.refelem import RefElem
from paper_1801_00246_b200 import meshgen


def _mesh(code=None, seed=11):
    tag = None if code is None else (lambda x, y: np.full(x.shape, code, dtype=np.int8))
    if code is None:
        tag = lambda x, y: np.where(x > 0.5, 1, 2).astype(np.int8)  # noqa: E731
    return meshgen.square(5, jitter=0.2, diag="random", order="morton", seed=seed, tag=tag)


@pytest.mark.parametrize("N", [1, 2, 4, 6])
def test_central_flux_gradient_and_divergence_are_negative_adjoints(N):
    """With central fluxes and the paired boundary mirrors the DG divergence is minus the adjoint of
    the DG gradient in the weak (mass-weighted) sense: sum_E (q, D u) = -sum_E (u, G q) for all q, u --
    interior faces cancel pairwise, velocity-Dirichlet faces (u+ = -u-, q+ = q-) and outflow faces
    (u+ = u-, q+ = -q-) cancel within themselves (derivation in DESIGN.md R20)."""
    m = _mesh()
    ref = RefElem(N)
    for axis in (0, 1):
        Wg = dgops.weak_derivative(m["VX"], m["VY"], m["EToV"], m["bc"], ref, axis, dgops.P_MIRROR)
        Wd = dgops.weak_derivative(m["VX"], m["VY"], m["EToV"], m["bc"], ref, axis, dgops.U_MIRROR)
        assert abs(Wd + Wg.T).max() <= 1e-12 * abs(Wg).max()
        assert abs(Wd - Wd.T).max() > 1e-3 * abs(Wd).max()  # not trivially symmetric


@pytest.mark.parametrize("N", [1, 2, 3, 5])
def test_gradient_exact_for_continuous_polynomials(N):
    """A globally continuous polynomial of degree <= N has no interior jumps; with p+ = p- on every
    boundary face (pressure Neumann, code 2) G p is its exact gradient at every node."""
    m = _mesh(code=2)
    ref = RefElem(N)
    x, y = physical_nodes(m["VX"], m["VY"], m["EToV"], ref)
    p = x ** N - 2 * x * y ** (N - 1) + 0.5 * y + 3.0
    gx, gy = dgops.dg_grad(m["VX"], m["VY"], m["EToV"], m["bc"], ref, p)
    ex = N * x ** (N - 1) - 2 * y ** (N - 1)
    ey = -2 * (N - 1) * x * y ** max(N - 2, 0) + 0.5
    assert np.abs(gx - ex).max() <= 1e-10 and np.abs(gy - ey).max() <= 1e-10


@pytest.mark.parametrize("N", [1, 2, 4])
def test_divergence_exact_for_continuous_polynomials(N):
    """With u+ = u- on every boundary face (code 1) D u is the exact divergence of a continuous u."""
    m = _mesh(code=1)
    ref = RefElem(N)
    x, y = physical_nodes(m["VX"], m["VY"], m["EToV"], ref)
    ux, uy = x ** N + y, x * y ** (N - 1) - 2.0
    d = dgops.dg_div(m["VX"], m["VY"], m["EToV"], m["bc"], ref, ux, uy)
    ex = N * x ** (N - 1) + (N - 1) * x * y ** max(N - 2, 0)
    assert np.abs(d - ex).max() <= 1e-10


def test_boundary_jumps_follow_the_paper():
    """Constant p = 1: on an outflow (pressure Dirichlet) face p* = 0, so G 1 = 1/2 sum_f (sJ/J) LIFT_f
    n (-2) != 0 near it; with pressure-Neumann faces only, G 1 = 0."""
    ref = RefElem(2)
    for code, zero in ((2, True), (1, False)):
        m = _mesh(code=code)
        gx, gy = dgops.dg_grad(m["VX"], m["VY"], m["EToV"], m["bc"], ref, np.ones(m["EToV"].shape[0] * ref.Np))
        assert (max(np.abs(gx).max(), np.abs(gy).max()) <= 1e-11) == zero


@pytest.mark.parametrize("N", [1, 3, 5])
def test_quadrature_route_matches_lift_route(N):
    """Two independent oracle routes for G p: the variational form by quadrature (basis evaluated at
    physical points, no lift) and the strong form with Dr, Ds and the lift."""
    m = _mesh(seed=12)
    ref = RefElem(N)
    p = meshgen.uniform_field(m["EToV"].shape[0], ref.Np, seed=7)
    a = dgops.dg_grad(m["VX"], m["VY"], m["EToV"], m["bc"], ref, p)
    b = dgops.nodal_grad_lift(m["VX"], m["VY"], m["EToV"], m["bc"], ref, p)
    for u, v in zip(a, b):
        assert np.abs(u - v).max() <= 1e-11 * np.abs(v).max()
