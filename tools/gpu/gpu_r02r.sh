#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02r; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_a_kernels.py -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_configs.py -k "A or C" -x -q > $O/pytest_cfg.log 2>&1; echo "exit $?" >> $O/pytest_cfg.log
ORDER=7 timeout 600 python tools/eval_ab.py NONE x > $O/eval_C.txt 2>&1
timeout 600 python tools/eval_ab.py NONE x > $O/eval_B.txt 2>&1
tail -2 $O/pytest.log $O/pytest_cfg.log; cat $O/eval_*.txt
