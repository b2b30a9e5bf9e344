import os, sys, subprocess
sys.path.insert(0, os.getcwd())
import paper_1801_00246_b200._lib as L
L.LIB_PATH = sys.argv[1]
import torch
from paper_1801_00246_b200 import Ipdg, meshgen
mesh = meshgen.square(707, jitter=0.2, diag="random", order="morton", seed=3)
for N in (1, 2, 3):
    for v in (3, 5):
        op = Ipdg(N, mesh); op.set_variant(v)
        us = [torch.rand(op.K, op.Np, dtype=torch.float64, device="cuda") for _ in range(6)]
        o = [torch.empty_like(us[0]) for _ in range(6)]
        for i in range(3): op.ax(us[i % 6], o[i % 6])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(50): op.ax(us[i % 6], o[i % 6])
        e1.record(); torch.cuda.synchronize()
        print(os.path.basename(sys.argv[1]), "N", N, "variant", v, "%.1f us" % (e0.elapsed_time(e1) / 50 * 1e3))
