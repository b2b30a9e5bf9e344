"""Partitioned Ax on one GPU (SURVEY T4'): P contexts hold the partitions of one mesh, their halo
rows are packed by the library (ipdg_halo_pack) and installed in the neighbours' ghost buffers
(ipdg_halo_set) instead of going through NCCL; the gathered result must equal the
single-context Ax (same per-element arithmetic) and the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.assemble import assemble  # noqa: E402
from oracle.refelem import RefElem  # noqa: E402
from paper_1801_00246_b200 import Ipdg, IpdgError, meshgen, partition  # noqa: E402


def _mesh():
    return meshgen.square(14, jitter=0.2, diag="random", order="morton", seed=12,
                          tag=lambda x, y: np.where(y > 0.4, 1, 2).astype(np.int8))


@pytest.mark.parametrize("N,variant", [(1, 1), (4, 1), (6, 1), (8, 1), (1, 2), (4, 2), (6, 2), (8, 2), (2, 4), (4, 4), (6, 4), (1, 5), (2, 5), (1, 6), (3, 6), (4, 6), (8, 6)])
@pytest.mark.parametrize("P", [2, 3])
def test_partitioned_ax_loopback(N, P, variant):
    m = _mesh()
    part = meshgen.rcb_partition(m["VX"], m["VY"], m["EToV"], P)
    ranks = partition.split(m, part, P)
    ops = [Ipdg.from_rank_mesh(N, rm) for rm in ranks]
    for op in ops:
        op.set_variant(variant)
    Np = ops[0].Np
    u = meshgen.uniform_field(m["EToV"].shape[0], Np, 100 + N)
    uloc = [torch.from_numpy(u[rm.elems]).cuda() for rm in ranks]
    sends = [op.halo_pack(ul) for op, ul in zip(ops, uloc)]
    for rm, op in zip(ranks, ops):
        ghosts = torch.zeros(max(rm.H, 1), Np, dtype=torch.float64, device="cuda")
        for j, q in enumerate(rm.nbr_ranks):
            src = ranks[int(q)]
            jj = int(np.nonzero(src.nbr_ranks == rm.rank)[0][0])
            ghosts[rm.recv_off[j]:rm.recv_off[j + 1]] = sends[int(q)][src.send_off[jj]:src.send_off[jj + 1]]
        op.halo_set(ghosts)
    Au = np.zeros_like(u)
    for rm, op, ul in zip(ranks, ops, uloc):
        Au[rm.elems] = op.ax(ul).cpu().numpy()
    gop = Ipdg(N, m)
    gop.set_variant(variant)
    ref = gop.ax(torch.from_numpy(u).cuda()).cpu().numpy()
    assert np.abs(Au - ref).max() <= 1e-14 * np.abs(ref).max()
    A = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], RefElem(N))
    Ao = A @ u.ravel()
    assert np.linalg.norm(Au.ravel() - Ao) <= 1e-12 * np.linalg.norm(Ao)
    # Jacobi diagonal across remote faces (tau uses the ghost's geometry)
    for rm, op in zip(ranks, ops):
        d = op.diag().cpu().numpy()
        dg = A.diagonal().reshape(-1, Np)[rm.elems]
        assert np.abs(d - dg).max() <= 1e-12 * np.abs(dg).max()


def test_distributed_pcg_needs_communicator():
    m = _mesh()
    part = meshgen.rcb_partition(m["VX"], m["VY"], m["EToV"], 2)
    rm = partition.split(m, part, 2, ranks=[0])[0]
    op = Ipdg.from_rank_mesh(3, rm)
    b = torch.ones(op.K, op.Np, dtype=torch.float64, device="cuda")
    with pytest.raises(IpdgError):
        op.pcg_solve(b, tol=1e-8, maxit=10)
