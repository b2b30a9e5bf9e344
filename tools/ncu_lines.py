"""Aggregate an ncu source page (cuda,sass csv) per CUDA source line: stall samples + instructions."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
agg = defaultdict(lambda: [0.0, 0.0, ""])
stall_cols = []
per_stall = defaultdict(float)
for r in rows:
    if len(r) > 5 and r[0] == "Line No":
        hdr = r
        idx = {h: j for j, h in enumerate(hdr)}
        stall_cols = [(h, j) for j, h in enumerate(hdr) if h.startswith("stall_")]
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0] not in ("-", ""):
        ln = r[0]
        s = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        ie = float(r[idx["Instructions Executed"]] or 0)
        agg[ln][0] += s
        agg[ln][1] += ie
        agg[ln][2] = r[1][:100]
        for h, j in stall_cols:
            try:
                per_stall[h] += float(r[j] or 0)
            except ValueError:
                pass
tot = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
print("total samples %.0f, instructions %.0f" % (tot, tot_i))
for ln, (s, ie, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print("%5.1f%% samp %5.1f%% inst  L%-4s %s" % (100 * s / tot, 100 * ie / tot_i, ln, src))
print("stall reasons:")
st = sum(per_stall.values()) or 1
for h, v in sorted(per_stall.items(), key=lambda kv: -kv[1])[:12]:
    print("  %-28s %5.1f%%" % (h, 100 * v / st))
