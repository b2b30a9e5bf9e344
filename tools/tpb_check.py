"""Quick parity + timing check of one kernel variant against the oracle (small meshes) and against the
auto variant (C2 timing).  usage: python tools/tpb_check.py [--variant 6] [--Ns 1 2 3 4 5] [--time]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import solvers  # noqa: E402
from oracle.assemble import assemble, mass_matrix  # noqa: E402
from oracle.refelem import RefElem  # noqa: E402
from paper_1801_00246_b200 import Ipdg, meshgen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--variant", type=int, default=6)
ap.add_argument("--Ns", type=int, nargs="+", default=[1, 2, 3, 4, 5])
ap.add_argument("--time", action="store_true")
ap.add_argument("--only", action="store_true", help="time only the chosen variant")
ap.add_argument("--noparity", action="store_true")
a = ap.parse_args()


def tag(x, y):
    return np.where(y < 0.5, 1, 2).astype(np.int8)


m = meshgen.square(14, jitter=0.2, diag="random", order="morton", seed=31, tag=tag)  # K = 392: 4 blocks
for N in ([] if a.noparity else a.Ns):
    ref = RefElem(N)
    A0 = assemble(m["VX"], m["VY"], m["EToV"], m["bc"], ref)
    Mg = mass_matrix(m["VX"], m["VY"], m["EToV"], ref)
    op = Ipdg(N, m)
    op.set_variant(a.variant)
    out = {"N": N, "variant": a.variant, "kernel": op.info()["kernel"]}
    for lam in (0.0, 0.7):
        u = meshgen.uniform_field(op.K, op.Np, seed=500 + N)
        Au = op.ax(torch.from_numpy(u).cuda(), lam=lam).cpu().numpy()
        r = ((A0 + lam * Mg) @ u.ravel()).reshape(Au.shape)
        out["ax_err_lam%g" % lam] = float(np.linalg.norm(Au - r) / np.linalg.norm(r))
    b = solvers.rhs_mass_interp(m["VX"], m["VY"], m["EToV"], ref, lambda x, y: np.exp(-((x - 0.3) ** 2 + y ** 2) / 0.1)).ravel()
    for pc in (0, 1):
        x, st = op.pcg_solve(torch.from_numpy(b.reshape(op.K, op.Np)).cuda(), precond=pc, tol=1e-9, maxit=20000)
        D = A0.diagonal()
        _, sto = solvers.pcg(lambda v: A0 @ v, b, 1e-9, 20000, (1.0 / D) if pc else None)
        res = np.linalg.norm(b - A0 @ x.cpu().numpy().ravel()) / np.linalg.norm(b)
        out["pcg%d" % pc] = [st["iterations"], sto["iterations"], float(res)]
    print(json.dumps(out), flush=True)

if a.time:
    stream = torch.cuda.current_stream()
    for N in a.Ns:
        mesh = meshgen.square(316, jitter=0.2, diag="random", order="morton", seed=2)
        for v in ((0, a.variant) if not a.only else (a.variant,)):
            op = Ipdg(N, mesh)
            op.set_variant(v)
            K, Np = op.K, op.Np
            nbuf = 6
            us = [torch.rand(K, Np, dtype=torch.float64, device="cuda") for _ in range(nbuf)]
            outs = [torch.empty_like(us[0]) for _ in range(nbuf)]
            for i in range(3):
                op.ax(us[i % nbuf], outs[i % nbuf])
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 50
            e0.record(stream)
            for i in range(n):
                op.ax(us[i % nbuf], outs[i % nbuf])
            e1.record(stream)
            torch.cuda.synchronize()
            ax_us = 1e3 * e0.elapsed_time(e1) / n
            bb = op.mass(us[0])
            x = torch.zeros_like(bb)
            ma = mb = float("nan")
            try:
                op.pcg_begin(bb, x, precond=1, tol=0.0)
                op.pcg_iterate(5)
                ma, mb = op.pcg_iterate_profiled(200)
                op.pcg_end()
            except Exception as ex:  # noqa: BLE001  (ablation builds break the solve)
                print("pcg:", str(ex)[:80])
            print(json.dumps({"C2": True, "N": N, "variant": v, "kernel": op.info()["kernel"], "ax_us": round(ax_us, 2),
                              "pass_a_us": round(1e3 * ma / 200, 2), "pass_b_us": round(1e3 * mb / 200, 2)}), flush=True)
            del us, outs, op
            torch.cuda.empty_cache()
