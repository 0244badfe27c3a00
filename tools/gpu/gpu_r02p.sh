#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02p; mkdir -p $O
timeout 300 python tools/trace_probe.py > $O/trace.txt 2>&1
timeout 900 python tools/eval_ab.py FMMGPU_MU_KEEP_SMS 0 4 8 16 24 32 > $O/ab_keep.txt 2>&1
cat $O/ab_keep.txt; tail -40 $O/trace.txt
