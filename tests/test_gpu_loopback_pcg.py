"""Distributed PCG on one GPU (SURVEY T4'; P:219 PCG over P:382's element partition): P = 2, 3 contexts
hold the RCB partitions of one mesh and run the library's distributed iteration in lockstep
(ipdg_loopback_pcg_solve): p_k packed at the send rows with pass A's decisions (k_pack_p), the halo
exchanged by device copies in the plans' order, pass A over interior then halo-boundary blocks with the
two-part p.Ap reduction, pass B, and fixed-order sums in place of the NCCL all-reduces.  Only the
transport differs from the NCCL path.

Bars (BASELINE.json north_star): iterations within +-1 of the oracle's textbook PCG on the assembled
global operator, widened only by the oracle's own spread under reorderings of the unknowns (DESIGN.md
R15); the oracle-computed residual of the gathered GPU solution <= tol (1 + 1e-6), or within the range of
true residuals the oracle's own solves reach under those reorderings, widened by that range's width as the
iteration bar is (the recursive residual stops at tol, the true one drifts by rounding; the partitioned
sums are one more such ordering).
"""
import functools

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import solvers  # noqa: E402
from oracle.assemble import assemble  # noqa: E402
from oracle.refelem import RefElem  # noqa: E402
from paper_1801_00246_b200 import Ipdg, loopback_pcg_solve, meshgen, partition  # noqa: E402
from pcg_spread import check_iterations, oracle_iteration_spread  # noqa: E402


def _mesh():
    return meshgen.square(14, jitter=0.2, diag="random", order="morton", seed=41,
                          tag=lambda x, y: np.where(y > 0.4, 1, 2).astype(np.int8))  # K = 392


@functools.lru_cache(maxsize=None)
def _problem(N, precond):
    m = _mesh()
    ref = RefElem(N)
    lam = 40.0 if precond == 2 else 0.0
    A = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], ref, lam=lam)
    b = solvers.rhs_mass_interp(m["VX"], m["VY"], m["EToV"], ref,
                                lambda x, y: np.exp(-((x - 0.3) ** 2 + y ** 2) / 0.1)).ravel()
    tol = 1e-9
    trues = []
    xo, st, counts = oracle_iteration_spread(A, b, tol, 20000, precond, lam, ref, m, true_res=trues)
    true_o = max(trues) + (max(trues) - min(trues))
    return m, A, b, lam, tol, st["iterations"], tuple(counts), true_o


CASES = [(N, p, v) for N in (1, 3, 4, 6, 8) for p in (0, 1, 2) for v in (0, 4, 6)]


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("N,precond,variant", CASES)
def test_loopback_distributed_pcg(N, precond, variant, P):
    m, A, b, lam, tol, it_o, counts, true_o = _problem(N, precond)
    part = meshgen.rcb_partition(m["VX"], m["VY"], m["EToV"], P)
    ranks = partition.split(m, part, P)
    ops = [Ipdg.from_rank_mesh(N, rm) for rm in ranks]
    for op in ops:
        op.set_variant(variant)
    Np = ops[0].Np
    bg = b.reshape(-1, Np)
    bs = [torch.from_numpy(np.ascontiguousarray(bg[rm.elems])).cuda() for rm in ranks]
    xs = [torch.zeros_like(bl) for bl in bs]
    st = loopback_pcg_solve(ops, bs, xs, lam=lam, precond=precond, tol=tol, maxit=20000)
    its = {s["iterations"] for s in st}
    assert len(its) == 1, st  # every partition stops at the same iteration (identical reduced scalars)
    assert all(s["status"] == 0 for s in st)
    check_iterations(st[0]["iterations"], it_o, counts)
    x = np.zeros_like(bg)
    for rm, xl in zip(ranks, xs):
        x[rm.elems] = xl.cpu().numpy()
    r = np.linalg.norm(b - A @ x.ravel()) / np.linalg.norm(b)
    assert r <= max(tol, true_o) * (1 + 1e-6), (r, true_o)


def test_loopback_split_pass_a_is_active():
    """The partitions have halo-boundary blocks, so pass A runs as two launches with the two-part
    p.Ap reduction (the overlapped NCCL schedule's kernel sequence)."""
    m = _mesh()
    part = meshgen.rcb_partition(m["VX"], m["VY"], m["EToV"], 2)
    rm = partition.split(m, part, 2)[0]
    op = Ipdg.from_rank_mesh(4, rm)
    S, H = op.halo_info()
    assert S > 0 and H > 0
