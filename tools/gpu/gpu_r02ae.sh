#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ae; mkdir -p $O
timeout 2400 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python tools/scratch/sanitize_probe.py > $O/memcheck.txt 2>&1; echo "exit $?" >> $O/memcheck.txt
timeout 1800 compute-sanitizer --tool racecheck --print-limit 20 python tools/scratch/sanitize_probe.py > $O/racecheck.txt 2>&1; echo "exit $?" >> $O/racecheck.txt
tail -15 $O/memcheck.txt; tail -15 $O/racecheck.txt
