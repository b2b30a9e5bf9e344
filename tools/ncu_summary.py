"""Summarise an ncu --set full capture of k_sipdg into profiles/ (JSON + markdown).

usage: python tools/ncu_summary.py gpurun_out/prof_X.ncu-rep profiles/r01_ncu_X [--N 4 --K 199712]
Writes <out>.json / <out>.md and updates profiles/ncu_summary.json (read by bench.py for
roofline.traffic) with the pass-A (k_sipdg<N,1,*>) DRAM bytes per launch.
"""
import argparse
import csv
import io
import json
import os
import subprocess

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dmma_pipe_pct": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smem_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "ipc": "sm__inst_executed.sum.per_cycle_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "dyn_smem_bytes": "launch__shared_mem_per_block_dynamic",
    "grid": "launch__grid_size",
    "dram_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_bytes": "lts__t_bytes.sum",
}
SCALE = {"Kbyte/block": 1e3, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "us": 1.0, "ms": 1e3, "ns": 1e-3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--N", type=int, default=4)
    ap.add_argument("--K", type=int, default=199712)
    ap.add_argument("--iteration", type=int, default=None, help="PCG iteration of the captured pass-A launch")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: j for j, h in enumerate(hdr)}
    out = []
    for r in rows[2:]:
        d = {"kernel": r[idx["Kernel Name"]], "id": r[idx["ID"]]}
        for k, m in KEYS.items():
            if m in idx:
                v = r[idx[m]].replace(",", "")
                try:
                    v = float(v) * SCALE.get(units[idx[m]], 1.0)
                except ValueError:
                    pass
                d[k] = v
        if "dram_read_bytes" in d and "dram_write_bytes" in d:
            d["dram_bytes"] = d["dram_read_bytes"] + d["dram_write_bytes"]
        st = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(r[j].replace(",", "") or 0)
              for h, j in idx.items() if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
        tot = sum(st.values()) or 1.0
        d["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]}
        out.append(d)
    json.dump({"source": os.path.basename(a.rep), "N": a.N, "K": a.K, "launches": out}, open(a.out + ".json", "w"), indent=1)
    with open(a.out + ".md", "w") as f:
        f.write("| id | kernel | us | DRAM MB | DMMA pipe % | FP64 pipe % | smem wf % | bank conflicts | IPC | regs | smem KB |\n|---|---|---|---|---|---|---|---|---|---|---|\n")
        for d in out:
            f.write("| %s | %s | %.1f | %.1f | %.1f | %.1f | %.1f | %.2e | %.0f | %d | %.1f |\n" % (
                d["id"], d["kernel"][:40], d.get("duration_us", 0), d.get("dram_bytes", 0) / 1e6, d.get("dmma_pipe_pct", 0),
                d.get("fp64_pipe_pct", 0), d.get("smem_pct", 0), d.get("smem_bank_conflicts", 0), d.get("ipc", 0),
                int(d.get("registers", 0)), d.get("dyn_smem_bytes", 0) / 1e3))
        f.write("\nWarp-state samples (% of all samples):\n\n")
        for d in out:
            f.write("- %s %s: %s\n" % (d["id"], d["kernel"][:40], ", ".join("%s %.1f" % kv for kv in d["stall_pct"].items())))
    def kname(d):
        return d["kernel"].split("<")[0].split()[-1].split("::")[-1]
    pa = [d for d in out if ("<%d, 1" % a.N) in d["kernel"] and kname(d) in ("k_sipdg", "k_pipe", "k_tpb", "k_gather")]
    summ_path = os.path.join(os.path.dirname(a.out), "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    if pa:
        summ["pass_a"] = {"N": a.N, "K": a.K, "kernel": kname(pa[0]), "dram_bytes_per_launch": pa[0].get("dram_bytes"),
                          "duration_us_under_ncu": pa[0].get("duration_us"), "source": os.path.basename(a.rep),
                          "pcg_iteration": a.iteration}
    ax = [d for d in out if ("<%d, 0" % a.N) in d["kernel"] and kname(d) in ("k_sipdg", "k_pipe", "k_tpb", "k_gather")]
    if ax:
        summ["ax"] = {"N": a.N, "K": a.K, "kernel": kname(ax[0]), "dram_bytes_per_launch": ax[0].get("dram_bytes"),
                      "duration_us_under_ncu": ax[0].get("duration_us"), "source": os.path.basename(a.rep)}
    json.dump(summ, open(summ_path, "w"), indent=1)
    print(open(a.out + ".md").read())


if __name__ == "__main__":
    main()
