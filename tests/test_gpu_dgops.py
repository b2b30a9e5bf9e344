"""GPU parity of the DG gradient / divergence with central fluxes (Eqs. INS_SD_4_1,
INS_SD_4_2) against the oracle (quadrature route, oracle/dgops.py), element-wise."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import dgops  # noqa: E402
from oracle.refelem import RefElem  # noqa: E402
from paper_1801_00246_b200 import Ipdg, meshgen  # noqa: E402

TOL = 1e-12


def gpu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


MESHES = {
    "mixed": lambda: meshgen.square(9, jitter=0.2, diag="random", order="morton", seed=31,
                                    tag=lambda x, y: np.where(x > 0.7, 1, 2).astype(np.int8)),
    "cylinder_like": lambda: meshgen.square(7, jitter=0.15, diag="random", order="random", seed=32,
                                            tag=lambda x, y: np.where(y < 0.2, 1, 2).astype(np.int8)),
}


@pytest.mark.parametrize("N", list(range(1, 9)))
@pytest.mark.parametrize("mesh", sorted(MESHES))
def test_dg_grad_and_div_match_oracle(N, mesh):
    m = MESHES[mesh]()
    ref = RefElem(N)
    op = Ipdg(N, m)
    K = op.K
    p = meshgen.uniform_field(K, op.Np, seed=40 + N)
    ux = meshgen.uniform_field(K, op.Np, seed=50 + N)
    uy = meshgen.uniform_field(K, op.Np, seed=60 + N)
    gx, gy = op.dg_grad(gpu(p))
    d = op.dg_div(gpu(ux), gpu(uy))
    ox, oy = dgops.dg_grad(m["VX"], m["VY"], m["EToV"], m["bc"], ref, p)
    od = dgops.dg_div(m["VX"], m["VY"], m["EToV"], m["bc"], ref, ux, uy)
    for a, b in ((gx, ox), (gy, oy), (d, od)):
        a = a.cpu().numpy()
        assert rel(a.ravel(), b.ravel()) <= TOL, (N, mesh)
        err = np.abs(a - b).max(axis=1) / np.maximum(np.abs(b).max(axis=1), 1e-300)
        assert err.max() <= 1e-10


def test_dg_ops_ragged_chunks_and_errors():
    """K not a multiple of the per-CTA chunk; bad arguments are loud."""
    m = meshgen.square(3, jitter=0.1, diag="random", seed=5)  # K = 18
    op = Ipdg(5, m)
    p = gpu(meshgen.uniform_field(op.K, op.Np, seed=1))
    gx, gy = op.dg_grad(p)
    ox, oy = dgops.dg_grad(m["VX"], m["VY"], m["EToV"], m["bc"], RefElem(5), p.cpu().numpy())
    assert rel(gx.cpu().numpy().ravel(), ox.ravel()) <= TOL and rel(gy.cpu().numpy().ravel(), oy.ravel()) <= TOL
    from paper_1801_00246_b200 import _lib
    L = _lib.lib()
    assert L.ipdg_dg_grad(op.ctx, p.data_ptr(), p.data_ptr(), gy.data_ptr(), None) == _lib.IPDG_EINVAL
    assert L.ipdg_dg_div(op.ctx, p.data_ptr(), gx.data_ptr(), p.data_ptr(), None) == _lib.IPDG_EINVAL
    assert L.ipdg_dg_grad(op.ctx, None, gx.data_ptr(), gy.data_ptr(), None) == _lib.IPDG_EINVAL
