#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02e
cap() {  # name regex skip args...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$rx" -s "$skip" -c 1 \
    -o "gpurun_out/r02e/$name" -f python tools/profile_eval.py "$@" > "gpurun_out/r02e/$name.out" 2>&1
  python tools/ncu_summary.py "gpurun_out/r02e/$name.ncu-rep" > "gpurun_out/r02e/$name.txt" 2>&1
}
cap D_ring 'k_p2p_mutual_ring' 0 20000000 8 5 1 ellipsoid
cap D_sub 'k_p2p_mutual<' 0 20000000 8 5 1 ellipsoid
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/r02e/D_launches.csv python tools/profile_eval.py 20000000 8 5 1 ellipsoid > /dev/null 2>&1
