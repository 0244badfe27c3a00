#!/bin/bash
# ncu full capture (with source) of P2M and the gather at config B
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bh; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_p2m_warp2" -c 1 -o $O/prof_p2m -f python tools/profile_eval.py 10000000 7 5 1 > $O/p2m.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_gather" -c 1 -o $O/prof_gather -f python tools/profile_eval.py 10000000 7 5 1 > $O/gather.out 2>&1
ls $O
