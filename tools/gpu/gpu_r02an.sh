#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02an; mkdir -p $O
timeout 900 python -m pytest tests/test_dist_input.py -x -q -k nccl -rs > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 600 python tools/eval_ab.py NONE x x > $O/eval_B.txt 2>&1
tail -15 $O/pytest.log; cat $O/eval_B.txt
