"""Small driver for ncu captures: a few Ax calls and PCG iterations at a BASELINE config."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1801_00246_b200 import Ipdg, meshgen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=4)
ap.add_argument("--nx", type=int, default=316)
ap.add_argument("--ax", type=int, default=3)
ap.add_argument("--pcg", type=int, default=3)
ap.add_argument("--variant", type=int, default=0)
ap.add_argument("--precond", type=int, default=1)
a = ap.parse_args()
mesh = meshgen.square(a.nx, jitter=0.2, diag="random", order="morton", seed=2)
op = Ipdg(a.N, mesh)
op.set_variant(a.variant)
u = torch.rand(op.K, op.Np, dtype=torch.float64, device="cuda")
for _ in range(a.ax):
    op.ax(u)
if a.pcg:
    b = op.mass(u)
    x = torch.zeros_like(b)
    op.pcg_begin(b, x, precond=a.precond, tol=0.0)
    op.pcg_iterate_profiled(a.pcg)
    op.pcg_end()
torch.cuda.synchronize()
print(op.info())
