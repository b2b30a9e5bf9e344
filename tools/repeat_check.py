"""Run the same Ax many times and report run-to-run differences (nondeterminism hunt)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1801_00246_b200 import Ipdg, meshgen  # noqa: E402

m = meshgen.square(15, jitter=0.2, diag="random", order="morton", seed=4, tag=lambda x, y: np.where(x < 0.5, 1, 2).astype(np.int8))
for N in [1, 4, 6]:
    for variant in (1, 2):
        op = Ipdg(N, m)
        op.set_variant(variant)
        u = torch.from_numpy(meshgen.uniform_field(op.K, op.Np, 200 + N)).cuda()
        ref = op.ax(u).clone()
        bad = 0
        for it in range(200):
            out = op.ax(u)
            if not torch.equal(out, ref):
                bad += 1
                d = (out - ref).abs()
                idx = torch.nonzero(d > 0)
                if bad <= 2:
                    print("N", N, "variant", variant, "iter", it, "ndiff", idx.shape[0], "max", d.max().item(), "elems", idx[:6, 0].tolist())
        print("N", N, "variant", variant, "mismatching runs", bad, flush=True)
