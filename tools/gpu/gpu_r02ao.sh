#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ao; mkdir -p $O
timeout 3000 compute-sanitizer --tool initcheck --print-limit 30 python tools/scratch/sanitize_probe.py > $O/initcheck.txt 2>&1; echo "exit $?" >> $O/initcheck.txt
true || timeout 1500 compute-sanitizer --tool synccheck --print-limit 30 python tools/scratch/sanitize_probe.py > $O/synccheck.txt 2>&1; echo "exit $?" >> $O/synccheck.txt
tail -40 $O/initcheck.txt; tail -8 $O/synccheck.txt
