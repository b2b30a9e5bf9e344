"""Per-source-line instructions executed per unit and warp-stall samples (top reasons) of an ncu source page.
usage: ncu -i rep --page source --csv --print-source cuda,sass [--launch-skip i --launch-count 1] > src.csv
       python tools/ncu_lines.py src.csv <units, e.g. elements>"""
import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
units=float(sys.argv[2])
fname="";hdr=None;out=[]
for r in rows:
    if len(r)==2 and r[0]=="File Path": fname=r[1].split('/')[-1]; continue
    if r and r[0]=="Line No": hdr=r; continue
    if hdr is None or len(r)<10 or r[0]=="" : continue
    d=dict(zip(hdr,r))
    try: n=int(d["Instructions Executed"]); s=int(d["Warp Stall Sampling (All Samples)"])
    except: continue
    st={k[6:]:int(v) for k,v in d.items() if k.startswith('stall_') and '(' not in k and v.isdigit() and int(v)>0}
    top=sorted(st.items(),key=lambda x:-x[1])[:3]
    out.append((fname,int(r[0]),n/units,s,top,r[1].strip()[:70]))
tot=sum(o[2] for o in out); ts=sum(o[3] for o in out)
print("instr/unit %.1f samples %d"%(tot,ts))
for o in out:
    if o[2]>=0.8 or o[3]>=ts*0.008:
        print("%-16s %4d %6.2f %5.1f%% %-40s %s"%(o[0],o[1],o[2],100*o[3]/ts,",".join("%s:%d"%t for t in o[4]),o[5]))
