"""Per-variant timing of Ax and PCG pass A / pass B (CUDA events, L2-defeating buffer rotation for Ax):
C2 (N = 4) and the C3 mesh for the requested degrees.  usage: python tools/variant_timing.py [--Ns 2 3 4 5] [--variants 4 6]"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1801_00246_b200 import Ipdg, meshgen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--Ns", type=int, nargs="+", default=[4])
ap.add_argument("--variants", type=int, nargs="+", default=[4, 6])
ap.add_argument("--mesh", default="C2")
ap.add_argument("--pcg", type=int, default=200)
a = ap.parse_args()
nx = 316 if a.mesh == "C2" else 707
mesh = meshgen.square(nx, jitter=0.2, diag="random", order="morton", seed=2 if a.mesh == "C2" else 3)
stream = torch.cuda.current_stream()
for N in a.Ns:
    for v in a.variants:
        op = Ipdg(N, mesh)
        try:
            op.set_variant(v)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"N": N, "variant": v, "error": str(e)}))
            continue
        K, Np = op.K, op.Np
        nbuf = max(2, int(math.ceil(4 * 126e6 / (2 * 8 * K * Np))))
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
        b = op.mass(us[0])
        x = torch.zeros_like(b)
        op.pcg_begin(b, x, precond=1, tol=0.0)
        op.pcg_iterate(5)
        ma, mb = op.pcg_iterate_profiled(a.pcg)
        op.pcg_end()
        info = op.info()
        print(json.dumps({"mesh": a.mesh, "N": N, "variant": v, "K": K, "ax_us": round(ax_us, 2),
                          "pass_a_us": round(1e3 * ma / a.pcg, 2), "pass_b_us": round(1e3 * mb / a.pcg, 2),
                          "kernel": info["kernel"], "smem": info["kernel_smem_bytes"], "grid": info["kernel_grid"]}), flush=True)
        del us, outs, op
        torch.cuda.empty_cache()
