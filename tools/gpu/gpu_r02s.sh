#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02s; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_a_kernels.py -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 600 python tools/eval_ab.py NONE x > $O/eval_B.txt 2>&1
N=20000000 H=8 DIST=ellipsoid timeout 600 python tools/eval_ab.py NONE x > $O/eval_D.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_p2p_mutual" -c 1 -o $O/B_p2p -f python tools/profile_eval.py 10000000 7 5 1 > $O/B_p2p.out 2>&1
tail -2 $O/pytest.log; cat $O/eval_*.txt
