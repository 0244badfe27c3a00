#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02d
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multigpu.py -x -q -k "p2p or deterministic or full_evaluation or multigpu or partition" > gpurun_out/r02d/pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02d/pytest.log
tail -5 gpurun_out/r02d/pytest.log
timeout 600 python tools/p2p_ab.py B 2>&1 | tee gpurun_out/r02d/ab_B.txt
timeout 600 python tools/p2p_ab.py D 2>&1 | tee gpurun_out/r02d/ab_D.txt
