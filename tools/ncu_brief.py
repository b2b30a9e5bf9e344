"""One-screen summary of every kernel in an ncu --set full report: duration, DRAM bytes, FP64/DMMA pipe,
warps active, instruction counts, stall reasons per issue, and the opcode mix by stall samples.
usage: python tools/ncu_brief.py gpurun_out/X.ncu-rep [--sass]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
KEYS = [("us", "gpu__time_duration.sum"), ("dram_rd_MB", "dram__bytes_read.sum"), ("dram_wr_MB", "dram__bytes_write.sum"),
        ("fp64%", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        ("dmma%", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
        ("warps_act", "sm__warps_active.avg.per_cycle_active"), ("regs", "launch__registers_per_thread"),
        ("inst", "smsp__inst_executed.sum"), ("smem%", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
        ("dram%", "dram__throughput.avg.pct_of_peak_sustained_elapsed")]
SC = {"Mbyte": 1, "Kbyte": 1e-3, "Gbyte": 1e3, "byte": 1e-6, "us": 1, "ms": 1e3, "ns": 1e-3}
for v in rows[2:]:
    name = v[h.index("Kernel Name")][:70]
    out = []
    for k, m in KEYS:
        if m in h:
            x = v[h.index(m)]
            try:
                x = float(x) * SC.get(units[h.index(m)], 1)
                out.append("%s=%.4g" % (k, x))
            except ValueError:
                pass
    print(name)
    print("  " + " ".join(out))
    st = []
    for i, n in enumerate(h):
        if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
            try:
                x = float(v[i])
            except ValueError:
                continue
            if x >= 0.05:
                st.append((x, n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    print("  stalls/issue: " + ", ".join("%s %.2f" % (n, x) for x, n in sorted(st, reverse=True)))
if "--sass" in sys.argv:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(src)))
    hdr = r[1]
    data = [x for x in r[2:] if len(x) >= len(hdr)]
    si, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    tot = sum(float(x[si] or 0) for x in data) or 1
    c, n = Counter(), Counter()
    for x in data:
        t = x[1].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        op = op.split(".")[0]
        c[op] += float(x[si] or 0)
        n[op] += float(x[ie] or 0)
    print("  opcode: samples% / executed warp-instructions")
    for k, s in c.most_common(14):
        print("   %-8s %5.1f%% %10d" % (k, 100 * s / tot, n[k]))
