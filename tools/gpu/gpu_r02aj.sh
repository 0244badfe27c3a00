#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02aj; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "near_block or tree_and_lists" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -k "A or H7 or B" > $O/pytest_cfg.log 2>&1; echo "exit $?" >> $O/pytest_cfg.log
for f in $O/pytest.log $O/pytest_cfg.log; do tail -3 $f; done
