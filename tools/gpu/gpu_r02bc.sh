#!/bin/bash
# memcheck + racecheck of every kernel family after the round-2 closing kernel changes
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bc; mkdir -p $O
timeout 2400 compute-sanitizer --tool memcheck --print-limit 30 python tools/scratch/sanitize_probe.py > $O/memcheck.txt 2>&1; echo "exit $?" >> $O/memcheck.txt
timeout 2400 compute-sanitizer --tool racecheck --print-limit 30 python tools/scratch/sanitize_probe.py > $O/racecheck.txt 2>&1; echo "exit $?" >> $O/racecheck.txt
tail -4 $O/memcheck.txt; tail -4 $O/racecheck.txt
