"""Per-iteration cost of PCG with the p-multigrid preconditioner (C2, N = 4): graph-replayed iterations vs
one V-cycle launched from the host, and the profiled split (pass A | pass B + V-cycle + r.z)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1801_00246_b200 import Ipdg, meshgen  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4
mesh = meshgen.square(316, jitter=0.2, diag="random", order="morton", seed=2)
op = Ipdg(N, mesh)
u = torch.rand(op.K, op.Np, dtype=torch.float64, device="cuda")
b = op.mass(u)
s = torch.cuda.current_stream()
for pc in (1, 3):
    x = torch.zeros_like(b)
    op.pcg_begin(b, x, precond=pc, tol=0.0)
    op.pcg_iterate(4)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    op.pcg_iterate(64)
    e1.record(s)
    torch.cuda.synchronize()
    graph_ms = e0.elapsed_time(e1) / 64
    ma, mb = op.pcg_iterate_profiled(16)
    op.pcg_end()
    r = torch.rand_like(b)
    op.pmg_apply(r)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(10):
        op.pmg_apply(r)
    e1.record(s)
    torch.cuda.synchronize()
    print(json.dumps({"N": N, "precond": pc, "graph_ms_per_iter": round(graph_ms, 4), "profiled_pass_a_ms": round(ma / 16, 4),
                      "profiled_pass_b_ms": round(mb / 16, 4), "vcycle_ms": round(e0.elapsed_time(e1) / 10, 4),
                      "launches_per_iter": None}), flush=True)
