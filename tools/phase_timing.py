"""Build a phase-timing copy of libipdg (-DIPDG_PHASE_TIMING) and report cycles per phase of k_sipdg (warp 0 of each CTA)."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1801_00246_b200 import build as B  # noqa: E402

out = "/tmp/libipdg_timing.so"
cmd = [B.NVCC] + B.FLAGS + B.nccl_flags()[0] + ["-DIPDG_PHASE_TIMING"] + [os.path.join(B.CSRC, x) for x in B.SOURCES] + ["-o", out] + B.nccl_flags()[1]
subprocess.run(cmd, check=True, capture_output=True)
import paper_1801_00246_b200._lib as L  # noqa: E402
L.LIB_PATH = out
import torch  # noqa: E402
from paper_1801_00246_b200 import Ipdg, meshgen  # noqa: E402

lib = L.lib()
fn = lib.ipdg_debug_phase_cycles
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 8)()
variant = int(os.environ.get("VARIANT", "1"))
names = (["top-wait", "P0 loads", "P1 grad", "P2 faces", "P3 gemm", "P3 store"] if variant == 1 else
         ["top-wait", "issue", "p/x stores", "P1+vol", "barrier", "P2/P3+store"])
for N in [int(a) for a in sys.argv[1:]] or [4]:
    mesh = meshgen.square(316, jitter=0.2, diag="random", order="morton", seed=2)
    op = Ipdg(N, mesh)
    op.set_variant(variant)
    u = torch.rand(op.K, op.Np, dtype=torch.float64, device="cuda")
    op.ax(u)
    torch.cuda.synchronize()
    fn(buf, 1)
    for mode in ("ax", "pcg"):
        if mode == "ax":
            for _ in range(10):
                op.ax(u)
        else:
            b = op.mass(u)
            x = torch.zeros_like(b)
            op.pcg_begin(b, x, precond=1, tol=0.0)
            op.pcg_iterate(10)
        torch.cuda.synchronize()
        fn(buf, 1)
        tot = sum(buf[:6])
        info = op.info()
        print("N=%d %s: grid %d, cycles per CTA per launch: %s" % (N, mode, info["grid"], ", ".join(
            "%s %.0f (%.0f%%)" % (names[i], buf[i] / 10 / info["grid"], 100 * buf[i] / tot) for i in range(6))))
        if mode == "pcg":
            op.pcg_end()
