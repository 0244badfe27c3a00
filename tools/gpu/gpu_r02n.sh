#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02n; mkdir -p $O
timeout 600 python tools/scratch/deep_diag.py > $O/deep_diag.txt 2>&1
timeout 600 python tools/scratch/deep_diag.py 12000 9 >> $O/deep_diag.txt 2>&1
cat $O/deep_diag.txt
