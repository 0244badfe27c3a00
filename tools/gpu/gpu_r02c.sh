#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02c
cap() {  # name regex skip args...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$rx" -s "$skip" -c 1 \
    -o "gpurun_out/r02c/$name" -f python tools/profile_eval.py "$@" > "gpurun_out/r02c/$name.out" 2>&1
  python tools/ncu_summary.py "gpurun_out/r02c/$name.ncu-rep" > "gpurun_out/r02c/$name.txt" 2>&1
}
cap B_mutual 'k_p2p_mutual' 0 10000000 7 5 1
cap B_drain 'k_p2p_drain' 0 10000000 7 5 1
cap D_mutual 'k_p2p_mutual' 0 20000000 8 5 1 ellipsoid
ls -la gpurun_out/r02c
