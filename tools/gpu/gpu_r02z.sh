#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02z; mkdir -p $O
FMMGPU_M2L_PA_STREAM=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "operators or full_evaluation or deterministic" > $O/pytest_s1.log 2>&1; echo "exit $?" >> $O/pytest_s1.log
timeout 900 python tools/eval_ab.py FMMGPU_M2L_PA_STREAM 0 1 2 3 > $O/ab_B.txt 2>&1
ORDER=7 timeout 900 python tools/eval_ab.py FMMGPU_M2L_PA_STREAM 0 1 2 3 > $O/ab_C.txt 2>&1
tail -2 $O/pytest_s1.log; cat $O/ab_*.txt
