"""Hot SASS instructions of an ncu source page (csv): samples, top stall reasons, instruction.
usage: ncu -i rep --page source --csv --print-source sass ... > src.csv; python tools/ncu_hot.py src.csv [n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
hdr, data = rows[1], [r for r in rows[2:] if len(r) >= len(rows[1])]
iS, iSrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[iS]) for r in data if r[iS].isdigit())
agg = {}
for r in data:
    for i in st:
        if r[i].isdigit():
            agg[hdr[i]] = agg.get(hdr[i], 0) + int(r[i])
print("total samples", tot, {k: round(100 * v / tot, 1) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]})
order = sorted(range(len(data)), key=lambda k: -int(data[k][iS]) if data[k][iS].isdigit() else 0)[:n]
for k in sorted(order):
    r = data[k]
    reasons = sorted(((int(r[i]), hdr[i][6:]) for i in st if r[i].isdigit() and int(r[i]) > 0), reverse=True)[:3]
    print("%5d %5s %-60s %s" % (k, r[iS], r[iSrc].strip()[:60], reasons))
