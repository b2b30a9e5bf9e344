import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1801_00246_b200 import Ipdg, meshgen
mesh = meshgen.square(316, jitter=0.2, diag="random", order="morton", seed=2)
for N in (1, 2, 3):
    for v in (4, 5):
        op = Ipdg(N, mesh); op.set_variant(v)
        u = torch.rand(op.K, op.Np, dtype=torch.float64, device="cuda")
        b = op.mass(u); x = torch.zeros_like(b)
        op.pcg_begin(b, x, precond=1, tol=0.0)
        op.pcg_iterate_profiled(5)
        ma, mb = op.pcg_iterate_profiled(100)
        op.pcg_end()
        print("N", N, "variant", v, "pass A %.2f us pass B %.2f us" % (10 * ma, 10 * mb))
