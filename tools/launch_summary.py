"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) per kernel: count, total, share."""
import csv
import io
import json
import sys
from collections import defaultdict

txt = open(sys.argv[1]).read()
start = txt.find('"ID"')
rows = list(csv.DictReader(io.StringIO(txt[start:])))
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0]
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3, "usecond": 1.0, "nsecond": 1e-3}.get(unit, 1.0)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
out = {k: {"launches": v[0], "total_us": round(v[1], 1), "avg_us": round(v[1] / v[0], 2), "share": round(v[1] / tot, 4)}
       for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}
print(json.dumps(out, indent=1))
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)
