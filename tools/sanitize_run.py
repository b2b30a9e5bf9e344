"""Small run of every kernel (all variants, Ax + PCG with point and block Jacobi, halo loopback, DG gradient /
divergence) for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1801_00246_b200 import Ipdg, meshgen, partition  # noqa: E402

m = meshgen.square(6, jitter=0.2, diag="random", order="morton", seed=3, tag=lambda x, y: np.where(x < 0.5, 1, 2).astype(np.int8))
for N in [int(a) for a in sys.argv[1:]] or [2, 6]:
    for variant in [v for v in (1, 2, 3, 4, 5) if v not in (3, 5) or N <= 4]:
        op = Ipdg(N, m)
        op.set_variant(variant)
        u = torch.from_numpy(meshgen.uniform_field(op.K, op.Np, 1)).cuda()
        op.ax(u)
        op.ax(u, lam=0.5)
        op.diag()
        b = op.mass(u)
        op.pcg_solve(b, precond=1, tol=1e-6, maxit=50)
        op.pcg_solve(b, precond=2, lam=10.0, tol=1e-6, maxit=50)
        op.dg_grad(u)
        op.dg_div(u, b)
        part = meshgen.rcb_partition(m["VX"], m["VY"], m["EToV"], 2)
        ranks = partition.split(m, part, 2)
        ops = [Ipdg.from_rank_mesh(N, rm) for rm in ranks]
        for o in ops:
            o.set_variant(variant)
        for rm, o in zip(ranks, ops):
            o.halo_set(torch.ones(max(rm.H, 1), o.Np, dtype=torch.float64, device="cuda"))
            o.ax(torch.from_numpy(u.cpu().numpy().reshape(-1, o.Np)[:0].copy()).cuda() if False else
                 torch.ones(o.K, o.Np, dtype=torch.float64, device="cuda"))
        torch.cuda.synchronize()
print("sanitize run done")
