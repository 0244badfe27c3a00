#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02am; mkdir -p $O
timeout 600 python tools/eval_ab.py NONE x x > $O/eval_B.txt 2>&1
N=20000000 H=8 DIST=ellipsoid timeout 900 python tools/eval_ab.py NONE x > $O/eval_D.txt 2>&1
timeout 600 python tools/scratch/rank_probe.py 8 > $O/rank8.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_multigpu.py tests/test_dist_input.py -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 1200 python -m pytest tests/test_gpu_configs.py -x -q -k "D or A" > $O/pytest_cfg.log 2>&1; echo "exit $?" >> $O/pytest_cfg.log
cat $O/eval_*.txt; head -1 $O/rank8.txt; for f in $O/pytest.log $O/pytest_cfg.log; do tail -2 $f; done
