"""Timing experiments: build a copy of libipdg with extra -D flags into /tmp and
report the C2 (N = 4) Ax and PCG pass A / pass B device times of the chosen variant.  Numbers only -- an
experiment flag may make the results wrong on purpose.
usage: python tools/exp_timing.py VARIANT [-DFLAG ...]  (flags: any compile-time switch under test)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1801_00246_b200 import build as B  # noqa: E402

variant = int(sys.argv[1])
flags = [f for f in sys.argv[2:] if f.startswith("-D")]
# a prebuilt library (tools/exp_build.sh) or build one now
out = os.path.join(ROOT, "exp_so", "libipdg_exp_%s.so" % "_".join(f[2:] for f in flags) if flags else "base")
if not os.path.exists(out):
    fl = [f for f in B.FLAGS if f not in ("-Xptxas", "-v")]
    cmd = [B.NVCC] + fl + B.nccl_flags()[0] + flags + [os.path.join(B.CSRC, x) for x in B.SOURCES] + ["-o", out] + B.nccl_flags()[1]
    subprocess.run(cmd, check=True, capture_output=True)
import paper_1801_00246_b200._lib as L  # noqa: E402
L.LIB_PATH = out
import torch  # noqa: E402
from paper_1801_00246_b200 import Ipdg, meshgen  # noqa: E402

mesh = meshgen.square(316, jitter=0.2, diag="random", order="morton", seed=2)
op = Ipdg(4, mesh)
op.set_variant(variant)
us = [torch.rand(op.K, op.Np, dtype=torch.float64, device="cuda") for _ in range(11)]
outs = [torch.empty_like(us[0]) for _ in range(11)]
for i in range(5):
    op.ax(us[i % 11], outs[i % 11])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(200):
    op.ax(us[i % 11], outs[i % 11])
e1.record()
torch.cuda.synchronize()
ax = e0.elapsed_time(e1) / 200
b = op.mass(us[0])
x = torch.zeros_like(b)
op.pcg_begin(b, x, precond=1, tol=0.0)
op.pcg_iterate_profiled(10)
ma, mb = op.pcg_iterate_profiled(100)
op.pcg_end()
print("variant %d %s: Ax %.2f us, pass A %.2f us, pass B %.2f us" % (variant, " ".join(flags) or "-", 1e3 * ax, 10 * ma, 10 * mb))
