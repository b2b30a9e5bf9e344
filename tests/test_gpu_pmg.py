"""GPU parity of the p-multigrid preconditioner (IPDG_PRECOND_PMG, DESIGN.md
R22-R26) against oracle/pmg.py: the power-iteration lmax of every level, one V-cycle element by element,
and PCG with the V-cycle as preconditioner (iterations within +-1 of the oracle's textbook PCG with the
oracle's V-cycle; residual of the GPU solution)."""
import functools

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import pmg, solvers  # noqa: E402
from paper_1801_00246_b200 import Ipdg, IpdgError, meshgen  # noqa: E402


def gpu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _mesh(nx=6):
    return meshgen.square(nx, jitter=0.2, diag="random", order="morton", seed=51,
                          tag=lambda x, y: np.where(y < 0.5, 1, 2).astype(np.int8))


@functools.lru_cache(maxsize=None)
def _hier(N, nx=6, lam=0.0):
    m = _mesh(nx)
    return m, pmg.PMG(m["VX"], m["VY"], m["EToV"], m["bc"], N, lam=lam)


@pytest.mark.parametrize("lam", [0.0, 3.0])
@pytest.mark.parametrize("N", range(1, 9))
def test_vcycle_matches_oracle(N, lam):
    m, H = _hier(N, lam=lam)
    op = Ipdg(N, m)
    r = meshgen.uniform_field(op.K, op.Np, seed=700 + N)
    z = op.pmg_apply(gpu(r), lam=lam).cpu().numpy().ravel()
    info = op.pmg_info()
    assert [d for d, _ in info] == H.degrees
    for (d, lm), lo in zip(info, H.lmax):
        assert abs(lm - lo) <= 1e-12 * lo, (d, lm, lo)
    zo = H.apply(r.ravel())
    assert np.linalg.norm(z - zo) <= 1e-12 * np.linalg.norm(zo)
    zr = zo.reshape(op.K, op.Np)
    err = np.abs(z.reshape(op.K, op.Np) - zr).max(axis=1) / np.maximum(np.abs(zr).max(axis=1), 1e-300)
    assert err.max() <= 1e-11


@pytest.mark.parametrize("variant", [0, 4, 6])
@pytest.mark.parametrize("N", [2, 3, 4, 6, 8])
def test_pmg_pcg_matches_oracle(N, variant):
    m, H = _hier(N, nx=8)
    A = H.A[0]
    b = solvers.rhs_mass_interp(m["VX"], m["VY"], m["EToV"], H.refs[0], meshgen.sin_sin_forcing).ravel()
    tol = 1e-9
    xo, sto = solvers.pcg(lambda v: A @ v, b, tol, 2000, apply_P=H.apply)
    op = Ipdg(N, m)
    op.set_variant(variant)
    x, st = op.pcg_solve(gpu(b.reshape(op.K, op.Np)), precond=3, tol=tol, maxit=2000)
    assert st["status"] == 0 and sto["status"] == 0
    assert abs(st["iterations"] - sto["iterations"]) <= 1, (st["iterations"], sto["iterations"])
    true_o = np.linalg.norm(b - A @ xo) / np.linalg.norm(b)
    r = np.linalg.norm(b - A @ x.cpu().numpy().ravel()) / np.linalg.norm(b)
    assert r <= max(tol, true_o) * (1 + 1e-3), (r, true_o)


def test_pmg_needs_one_partition():
    from paper_1801_00246_b200 import partition
    m = _mesh(8)
    part = meshgen.rcb_partition(m["VX"], m["VY"], m["EToV"], 2)
    rm = partition.split(m, part, 2, ranks=[0])[0]
    op = Ipdg.from_rank_mesh(3, rm)
    r = torch.ones(op.K, op.Np, dtype=torch.float64, device="cuda")
    with pytest.raises(IpdgError):
        op.pmg_apply(r)
