#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ah; mkdir -p $O
timeout 900 python tools/eval_ab.py FMMGPU_FUSE_DRAIN 0 1 0 1 > $O/ab_B.txt 2>&1
N=20000000 H=8 DIST=ellipsoid timeout 900 python tools/eval_ab.py FMMGPU_FUSE_DRAIN 0 1 > $O/ab_D.txt 2>&1
N=100000000 H=8 timeout 900 python tools/eval_ab.py FMMGPU_FUSE_DRAIN 0 1 > $O/ab_E.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_multigpu.py tests/test_dist_input.py tests/test_cpp_adapter.py -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q > $O/pytest_cfg.log 2>&1; echo "exit $?" >> $O/pytest_cfg.log
cat $O/ab_*.txt; for f in $O/pytest.log $O/pytest_cfg.log; do tail -2 $f; done
