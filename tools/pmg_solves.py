"""Full PCG solves to 1e-8 with point Jacobi and with the p-multigrid preconditioner (IPDG_PRECOND_PMG,
NEXT-3) on the BASELINE meshes, one GPU: iterations, solve time after a setup call (the Jacobi diagonal,
the pMG hierarchy and the iteration graphs are built once per operator), setup time.  JSON lines.
usage: python tools/pmg_solves.py [--configs C2 C4 C5] [--precond 1 3] [--maxit 400000]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1801_00246_b200 import Ipdg, meshgen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", nargs="+", default=["C2", "C4"])
ap.add_argument("--precond", type=int, nargs="+", default=[1, 3])
ap.add_argument("--maxit", type=int, default=400000)
ap.add_argument("--tol", type=float, default=1e-8)
a = ap.parse_args()

for cfg in a.configs:
    if cfg == "C2":
        N, mesh = 4, meshgen.square(316, jitter=0.2, diag="random", order="morton", seed=2)
        f = meshgen.sin_sin_forcing
    elif cfg == "C4":
        N, mesh = 6, meshgen.cylinder()
        f = None
    else:
        N = 8
        mesh, _ = meshgen.tiles(1414, 1, 1, jitter=0.2, seed=2)
        f = meshgen.sin_sin_forcing
    op = Ipdg(N, mesh)
    x, y = op.nodes()
    if f is None:  # SURVEY 8.4 / bench.py C4 right-hand side
        fv = torch.exp(-((x - 2.0) ** 2 + y ** 2) / 4.0)
    else:
        fv = torch.from_numpy(f(x.cpu().numpy(), y.cpu().numpy())).cuda()
    b = op.mass(fv.contiguous())
    for pc in a.precond:
        xs = torch.zeros_like(b)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        op.pcg_solve(b, x=xs, precond=pc, tol=a.tol, maxit=1)  # setup: Jacobi diagonal, pMG hierarchy, graphs
        torch.cuda.synchronize()
        setup = time.perf_counter() - t0
        xs = torch.zeros_like(b)
        t0 = time.perf_counter()
        xs, st = op.pcg_solve(b, x=xs, precond=pc, tol=a.tol, maxit=a.maxit)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        info = op.pmg_info() if pc == 3 else []
        print(json.dumps({"config": cfg, "N": N, "K": op.K, "dofs": op.K * op.Np, "precond": {1: "jacobi", 3: "pmg"}[pc],
                          "tol": a.tol, "iterations": st["iterations"], "rel_residual": st["rel_residual"],
                          "seconds": round(dt, 3), "setup_seconds": round(setup, 3),
                          "ms_per_iteration": round(1e3 * dt / max(1, st["iterations"]), 4),
                          "levels": [[d, round(l, 4)] for d, l in info]}), flush=True)
    del op
    torch.cuda.empty_cache()
