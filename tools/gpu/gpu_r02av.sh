#!/bin/bash
# pipelined e2e timeline at B with readback host/sync times; warm tree build time
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02av; mkdir -p $O
timeout 300 python tools/scratch/tree_time.py > $O/tree.log 2>&1
timeout 600 python tools/scratch/pipe_trace.py > $O/trace.log 2>&1
grep -v Warn $O/tree.log | tail -3
grep -v Warn $O/trace.log | tail -90
