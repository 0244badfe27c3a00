#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02w; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_dist_input.py tests/test_multigpu.py -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_configs.py -k "A or B or D" -x -q > $O/pytest_cfg.log 2>&1; echo "exit $?" >> $O/pytest_cfg.log
FMMGPU_TRACE=1 timeout 300 python tools/scratch/e2e_probe.py > $O/e2e_probe.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/tree_launches.csv python tools/scratch/profile_tree.py > $O/tree.out 2>&1
tail -2 $O/pytest.log $O/pytest_cfg.log; grep -v "alloc\]\|\[tree\]\|readback\|pipe\]" $O/e2e_probe.txt
