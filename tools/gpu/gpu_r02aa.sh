#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02aa; mkdir -p $O
ORDER=7 timeout 900 python tools/eval_ab.py FMMGPU_M2L_PA_STREAM 1 4 5 6 > $O/ab_C.txt 2>&1
ORDER=6 timeout 900 python tools/eval_ab.py FMMGPU_M2L_PA_STREAM 0 1 > $O/ab_l6.txt 2>&1
cat $O/ab_*.txt
