#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02m; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -k deep -q -rs -s > $O/pytest_deep.log 2>&1; echo "exit $?" >> $O/pytest_deep.log
ORDER=7 timeout 900 python tools/eval_ab.py FMMGPU_M2L_CLS_FAST 1 0 > $O/ab_clsfast_C.txt 2>&1
timeout 900 python tools/eval_ab.py FMMGPU_M2L_CLS_FAST 1 0 > $O/ab_clsfast_B.txt 2>&1
grep "deep tree" $O/pytest_deep.log; tail -2 $O/pytest_deep.log; cat $O/ab_*.txt
