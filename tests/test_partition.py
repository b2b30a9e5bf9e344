"""Multi-rank host logic (CPU): RCB partition, halo plans, and a world_size-2 gloo run of the
partitioned operator and the distributed PCG protocol with the oracle as the
local operator.  The CUDA side of the same plans is tested on one GPU in test_gpu_halo.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import solvers
from oracle.assemble import assemble
from oracle.mfree import MFree
from oracle.refelem import RefElem
from paper_1801_00246_b200 import meshgen, partition


def _mesh():
    return meshgen.square(9, jitter=0.2, diag="random", order="morton", seed=11,
                          tag=lambda x, y: np.where(x < 0.3, 1, 2).astype(np.int8))


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_rcb_partition_and_plans(P):
    m = _mesh()
    part = meshgen.rcb_partition(m["VX"], m["VY"], m["EToV"], P)
    counts = np.bincount(part, minlength=P)
    assert counts.sum() == m["EToV"].shape[0] and counts.max() - counts.min() <= 1
    ranks = partition.split(m, part, P)
    assert partition.check_plan(ranks)
    EToE, EToF = partition.global_connectivity(m["EToV"])
    for rm in ranks:
        cut = rm.bc == partition.REMOTE
        assert np.all((rm.remote >= 0) == cut)
        # every remote face points at the right ghost and face
        for e, f in zip(*np.nonzero(cut)):
            g = rm.ghosts[rm.remote[e, f]]
            assert EToE[rm.elems[e], f] == g and EToF[rm.elems[e], f] == rm.remote_face[e, f]
            assert part[g] != rm.rank
        # non-cut faces keep the global codes
        assert np.array_equal(rm.bc[~cut], m["bc"][rm.elems][~cut])


def extended_local(rm, m):
    """Own + ghost elements as one small mesh for the oracle (ghost outer faces: Neumann)."""
    ids = np.concatenate([rm.elems, rm.ghosts])
    sub = dict(VX=m["VX"], VY=m["VY"], EToV=m["EToV"][ids])
    EToE, _ = partition.global_connectivity(sub["EToV"])
    bc = np.where(EToE >= 0, 0, 2).astype(np.int8)
    own_bnd = (EToE[: rm.K] < 0)
    bc[: rm.K][own_bnd] = m["bc"][rm.elems][own_bnd]  # true physical codes on own faces
    sub["bc"] = bc
    return sub


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N = 3
    m = _mesh()
    part = meshgen.rcb_partition(m["VX"], m["VY"], m["EToV"], world)
    rm = partition.split(m, part, world, ranks=[rank])[0]
    ref = RefElem(N)
    sub = extended_local(rm, m)
    mf = MFree(sub["VX"], sub["VY"], sub["EToV"], sub["bc"], ref)
    Np = ref.Np

    def exchange(u_own):
        """Send the plan's rows, receive the ghost rows (one message per neighbour)."""
        ghosts = np.zeros((rm.H, Np))
        reqs, bufs = [], []
        for j, q in enumerate(rm.nbr_ranks):
            s = torch.from_numpy(np.ascontiguousarray(u_own[rm.send_elems[rm.send_off[j]:rm.send_off[j + 1]]]))
            r = torch.zeros(int(rm.recv_off[j + 1] - rm.recv_off[j]), Np, dtype=torch.float64)
            reqs.append(dist.isend(s, int(q)))
            reqs.append(dist.irecv(r, int(q)))
            bufs.append((j, r))
        for q in reqs:
            q.wait()
        for j, r in bufs:
            ghosts[rm.recv_off[j]:rm.recv_off[j + 1]] = r.numpy()
        return ghosts

    def apply(u_own):
        ext = np.concatenate([u_own, exchange(u_own)])
        return mf.apply(ext)[: rm.K]

    u = meshgen.uniform_field(m["EToV"].shape[0], Np, 5)  # global field, same on every rank
    Au_local = apply(u[rm.elems])

    def allreduce(x):
        t = torch.tensor(np.atleast_1d(x), dtype=torch.float64)
        dist.all_reduce(t)
        return t.numpy()

    # distributed Jacobi-PCG with the library's protocol: local dots + all-reduce of 1 and 2 doubles
    A_ext = assemble(sub["VX"], sub["VY"], sub["EToV"], sub["bc"], ref)
    d = A_ext.diagonal()[: rm.K * Np].reshape(rm.K, Np)  # own rows: complete (all neighbours present)
    f = lambda x, y: np.exp(-((x - 0.3) ** 2 + (y - 0.6) ** 2) / 0.05)  # noqa: E731
    b = solvers.rhs_mass_interp(m["VX"], m["VY"], m["EToV"][rm.elems], ref, f)
    x = np.zeros_like(b)
    r = b.copy()
    z = r / d
    p = z.copy()
    rho = allreduce(np.sum(r * z))[0]
    bb = allreduce(np.sum(b * b))[0]
    it = 0
    while it < 2000:
        q = apply(p)
        sigma = allreduce(np.sum(p * q))[0]
        alpha = rho / sigma
        x += alpha * p
        r -= alpha * q
        it += 1
        rz_rr = allreduce([np.sum(r * r / d), np.sum(r * r)])
        if rz_rr[1] <= 1e-10 ** 2 * bb:
            break
        beta = rz_rr[0] / rho
        rho = rz_rr[0]
        p = r / d + beta * p
    out[rank] = (rm.elems, Au_local, x, it)
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_world2_partitioned_operator_and_pcg():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    m = _mesh()
    N = 3
    ref = RefElem(N)
    A = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], ref)
    u = meshgen.uniform_field(m["EToV"].shape[0], ref.Np, 5)
    Au = (A @ u.ravel()).reshape(-1, ref.Np)
    f = lambda x, y: np.exp(-((x - 0.3) ** 2 + (y - 0.6) ** 2) / 0.05)  # noqa: E731
    b = solvers.rhs_mass_interp(m["VX"], m["VY"], m["EToV"], ref, f).ravel()
    xg, st = solvers.pcg(lambda v: A @ v, b, 1e-10, 2000, dinv=1.0 / A.diagonal())
    xg = xg.reshape(-1, ref.Np)
    for rank in range(world):
        elems, Au_local, x, it = out[rank]
        assert np.abs(Au_local - Au[elems]).max() <= 1e-12 * np.abs(Au).max()
        assert abs(it - st["iterations"]) <= 1
        assert np.abs(x - xg[elems]).max() <= 1e-8 * np.abs(xg).max()


@pytest.mark.parametrize("P", [2, 3, 5])
def test_rank_local_split_equals_global_split(P):
    """partition.split(..., ranks=[r]) builds rank r's connectivity from its own elements and their vertex
    neighbours only (no sort of the whole mesh); the plans must be identical to the global construction."""
    m = meshgen.square(15, jitter=0.2, diag="random", order="morton", seed=9,
                       tag=lambda x, y: np.where(y > 0.5, 1, 2).astype(np.int8))
    part = meshgen.rcb_partition(m["VX"], m["VY"], m["EToV"], P)
    full = partition.split(m, part, P)
    for r in range(P):
        loc = partition.split(m, part, P, ranks=[r])[0]
        ref = full[r]
        for name in ("elems", "EToV", "bc", "remote", "remote_face", "ghosts", "nbr_ranks", "send_off",
                     "send_elems", "recv_off"):
            assert np.array_equal(getattr(loc, name), getattr(ref, name)), (P, r, name)
