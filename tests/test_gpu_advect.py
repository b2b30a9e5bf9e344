"""GPU parity of the subcycling advection operator (ipdg_advect, NEXT-4; P:199-209 Eq. INS_CUB_N, Eq. KSS_3,
Alg. SSV / SSS; R27, R28) against oracle/advect.py, which integrates the variational form in
physical space with another exact rule (the library uses reference-space cubature operators)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import advect  # noqa: E402
from oracle.refelem import RefElem  # noqa: E402
from paper_1801_00246_b200 import Ipdg, IpdgError, meshgen, partition  # noqa: E402


def gpu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("bcs", ["mixed", "outflow"])
@pytest.mark.parametrize("N", range(1, 9))
def test_advect_matches_oracle(N, bcs):
    if bcs == "mixed":
        def tag(x, y):
            return np.where(y < 0.5, 1, 2).astype(np.int8)
    else:
        def tag(x, y):
            return np.ones_like(x, dtype=np.int8)
    m = meshgen.square(7, jitter=0.2, diag="random", order="morton", seed=61, tag=tag)  # K = 98: ragged last CTA
    ref = RefElem(N)
    op = Ipdg(N, m)
    K, Np = op.K, op.Np
    rng = np.random.default_rng(100 + N)
    f = [rng.uniform(-1, 1, (K, Np)) for _ in range(4)]
    Nu, Nv = op.advect(*(gpu(x) for x in f))
    ou, ov = advect.advection(m["VX"], m["VY"], m["EToV"], m["bc"], ref, *f)
    for g, o in ((Nu.cpu().numpy(), ou), (Nv.cpu().numpy(), ov)):
        assert np.linalg.norm(g - o) <= 1e-12 * np.linalg.norm(o)
        err = np.abs(g - o).max(axis=1) / np.maximum(np.abs(o).max(axis=1), 1e-300)
        assert err.max() <= 1e-11


def test_advect_rejects_partitions_and_aliasing():
    m = meshgen.square(6, jitter=0.2, diag="random", order="morton", seed=5)
    part = meshgen.rcb_partition(m["VX"], m["VY"], m["EToV"], 2)
    rm = partition.split(m, part, 2, ranks=[0])[0]
    op = Ipdg.from_rank_mesh(2, rm)
    x = torch.zeros(op.K, op.Np, dtype=torch.float64, device="cuda")
    with pytest.raises(IpdgError):
        op.advect(x, x, x, x)
