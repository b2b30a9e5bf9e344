import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle.assemble import assemble  # noqa: E402
from oracle.refelem import RefElem  # noqa: E402
from paper_1801_00246_b200 import Ipdg, meshgen  # noqa: E402

m = meshgen.square(15, jitter=0.2, diag="random", order="morton", seed=4, tag=lambda x, y: np.where(x < 0.5, 1, 2).astype(np.int8))
for N in (1, 6):
    ref = RefElem(N)
    A0 = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], ref)
    A1 = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], ref, lam=0.5)
    fails = 0
    for trial in range(40):
        op = Ipdg(N, m)
        op.set_variant(2)
        for lam, A in ((0.0, A0), (0.5, A1)):
            u = meshgen.uniform_field(op.K, op.Np, seed=200 + N)
            Au = op.ax(torch.from_numpy(u).cuda(), lam=lam).cpu().numpy()
            ref_ = A @ u.ravel()
            err = np.linalg.norm(Au.ravel() - ref_) / np.linalg.norm(ref_)
            if err > 1e-12:
                fails += 1
                d = np.abs(Au.ravel() - ref_).reshape(-1, op.Np).max(axis=1)
                bad = np.nonzero(d > 1e-10 * np.abs(ref_).max())[0]
                if fails <= 3:
                    print("N", N, "trial", trial, "lam", lam, "err %.3e" % err, "bad elems", bad[:10], "of", op.K, flush=True)
        del op
    print("N", N, "fails", fails, flush=True)
