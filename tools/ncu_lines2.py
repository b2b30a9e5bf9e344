"""Per-source-line totals (instructions executed per unit, stall samples) from
ncu --page source --csv --print-source cuda,sass.  usage: python tools/ncu_lines2.py src.csv units [min]"""
import csv
import sys

units = float(sys.argv[2])
mn = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
rows = list(csv.reader(open(sys.argv[1])))
fname = ""
out = []
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        iE = hdr.index("Instructions Executed")
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < len(hdr) or r[0] in ("", "Function Name"):
        continue
    n = int(r[iE]) if r[iE].isdigit() else 0
    s = int(r[iS]) if r[iS].isdigit() else 0
    out.append((fname, r[0], n / units, s, r[1].strip()[:90]))
tot = sum(o[2] for o in out)
tots = sum(o[3] for o in out)
print("total per unit %.1f, samples %d" % (tot, tots))
for o in out:
    if o[2] >= mn or o[3] >= tots * 0.01:
        print("%-18s %4s %6.2f %5d  %s" % o)
