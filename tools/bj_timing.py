"""Pass-A / pass-B device times of one PCG iteration with point Jacobi vs block-Jacobi (scaled inverse
mass) on the C2 recipe (N = 4) and a 300x300 square at N = 8 (screened Poisson, lambda = 1e3)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json  # noqa: E402

import torch  # noqa: E402

from paper_1801_00246_b200 import Ipdg, meshgen  # noqa: E402

for N, nx in ((4, 316), (8, 300)):
    mesh = meshgen.square(nx, jitter=0.2, diag="random", order="morton", seed=2)
    op = Ipdg(N, mesh)
    u = torch.rand(op.K, op.Np, dtype=torch.float64, device="cuda")
    b = op.mass(u)
    for pc in (1, 2):
        x = torch.zeros_like(b)
        op.pcg_begin(b, x, lam=1e3, precond=pc, tol=0.0)
        op.pcg_iterate_profiled(5)
        ma, mb = op.pcg_iterate_profiled(50)
        op.pcg_end()
        print(json.dumps({"N": N, "K": op.K, "precond": pc, "pass_a_us": round(1e3 * ma / 50, 2),
                          "pass_b_us": round(1e3 * mb / 50, 2), "pass_b_GBs_4vec": round(4 * 8 * op.K * op.Np / (mb / 50 / 1e3) / 1e9, 1)}))
