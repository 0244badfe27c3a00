#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02v; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/tree_launches.csv python tools/scratch/profile_tree.py > $O/tree.out 2>&1
python - <<'PY' > $O/tree_launches.txt
import csv
rows=list(csv.reader(open("gpurun_out/r02v/tree_launches.csv")))
hi=[i for i,r in enumerate(rows) if "Kernel Name" in r][0]
h=rows[hi]; ki,vi,ii=h.index("Kernel Name"),h.index("Metric Value"),h.index("ID")
data=[(r[ki],float(r[vi].replace(",",""))) for r in rows[hi+1:] if len(r)>vi]
half=len(data)//2
second=data[half:]
tot=sum(v for _,v in second)
print("launches", len(data), "second build", len(second), "sum ms", tot/1e6)
for k,v in second: print("%9.1f us  %s"%(v/1e3,k[:100]))
PY
head -80 $O/tree_launches.txt
