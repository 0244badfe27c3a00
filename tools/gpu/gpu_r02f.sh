#!/bin/bash
# re-entry pass: gpu tests + smoke, default bench, launch list, full capture of the mutual P2P at B
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02f; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -rs > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py --no-t1 > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_|Radix|Scan|RunLength|Reduce" --csv --log-file $O/launches.csv python tools/profile_eval.py 10000000 7 5 2 > $O/launches.out 2>&1
cap() {  # name regex skip
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$2" -s "$3" -c 1 -o $O/$1 -f python tools/profile_eval.py 10000000 7 5 1 > $O/$1.out 2>&1
  python tools/ncu_summary.py $O/$1.ncu-rep > $O/$1.txt 2>&1
}
cap B_p2p 'k_p2p_mutual' 0
cap B_m2la 'k_m2l_phase_a' 4
cap B_m2lb 'k_m2l_phase_b' 4
tail -3 $O/pytest_gpu.log; cat $O/smoke.log | tail -2; head -c 600 $O/bench.json
