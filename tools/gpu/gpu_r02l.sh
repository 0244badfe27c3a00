#!/bin/bash
# deep-tree test, launch lists of C and D, ncu of the P2P drain at B
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02l; mkdir -p $O/C $O/D $O/drain
timeout 900 python -m pytest tests/test_gpu_parity.py -k deep -x -q -rs > $O/pytest_deep.log 2>&1; echo "exit $?" >> $O/pytest_deep.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_|Radix|Scan|RunLength|Reduce" --csv --log-file $O/C/launches.csv python tools/profile_eval.py 10000000 7 7 2 > $O/C/launches.out 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_|Radix|Scan|RunLength|Reduce" --csv --log-file $O/D/launches.csv python tools/profile_eval.py 20000000 8 5 2 ellipsoid > $O/D/launches.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_p2p_drain" -c 1 -o $O/drain/B_drain -f python tools/profile_eval.py 10000000 7 5 1 > $O/drain/B_drain.out 2>&1
tail -3 $O/pytest_deep.log
