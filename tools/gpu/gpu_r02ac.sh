#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ac; mkdir -p $O
L="libfmmgpu.so libfmmgpu_b3s16.so libfmmgpu_b2s16.so libfmmgpu_bn128.so libfmmgpu_bn128s16.so"
ORDER=7 timeout 900 python tools/eval_ab.py FMMGPU_LIB $L > $O/ab_C.txt 2>&1
timeout 900 python tools/eval_ab.py FMMGPU_LIB $L > $O/ab_B.txt 2>&1
cat $O/ab_*.txt
