#!/bin/bash
# ncu --set full captures of the top kernels of one config-B evaluation (one per .ncu-rep):
# P2P, the leaf-level M2L phase A and phase B. usage: tools/ncu_top.sh [tag]
tag=${1:-r01}
mkdir -p gpurun_out
cap() {  # name regex skip
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" -s "$3" -c 1 \
    -o "gpurun_out/${tag}_$1" -f python tools/profile_eval.py 10000000 7 5 1 > "gpurun_out/${tag}_$1.out" 2>&1
}
cap p2p 'k_p2p' 0
cap m2la 'k_m2l_phase_a' 4
cap m2lb 'k_m2l_phase_b' 4
