"""Warp-stall samples per source line of an ncu report exported with
`ncu -i REP --page source --csv --print-source cuda,sass > x.csv`:
python tools/ncu_source_lines.py x.csv [top]. Produced profiles/r02_ncu_source_*.txt."""
import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
f=None; agg=[]; hdr=None
for r in rows:
    if len(r)>=2 and r[0]=='File Path': f=r[1].split('/')[-1]; continue
    if len(r)>3 and r[0]=='Line No': hdr=r; idx=[i for i,h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]; continue
    if hdr and len(r)>5 and r[0] not in ('',):
        try:
            st=sorted(((int(r[i]) if r[i] not in ('-','') else 0, hdr[i][6:]) for i in idx), reverse=True)[:4]
            agg.append((int(r[4]), r[7], f, r[0], r[1][:70], st))
        except Exception as e: pass
tot=sum(a[0] for a in agg)
for a in sorted(agg, reverse=True)[:int(sys.argv[2])]:
    print(f"{a[0]:7d} {100*a[0]/tot:5.1f}% {a[2]}:{a[3]} {a[4]}\n          "+", ".join(f"{n} {100*v/max(a[0],1):.0f}%" for v,n in a[5]))
