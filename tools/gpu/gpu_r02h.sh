#!/bin/bash
# distributed input tests + multi-GPU tests + P2P parity after the 12-warp change
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02h; mkdir -p $O
timeout 1200 python -m pytest tests/test_dist_input.py tests/test_multigpu.py -x -q -rs > $O/pytest_dist.log 2>&1; echo "exit $?" >> $O/pytest_dist.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $O/pytest_parity.log 2>&1; echo "exit $?" >> $O/pytest_parity.log
tail -5 $O/pytest_dist.log $O/pytest_parity.log
