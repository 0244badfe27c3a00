#!/bin/bash
# every BASELINE config through bench.py (same-config reference CPU baseline), current kernels
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02i; mkdir -p $O
nproc > $O/nproc.txt; free -g >> $O/nproc.txt
for cfg in A C D E; do
  timeout 1500 python bench.py --config $cfg --steps 10 --warmup 3 > $O/bench_$cfg.json 2> $O/bench_$cfg.err
done
for cfg in A C D E; do head -c 300 $O/bench_$cfg.json; echo; done
