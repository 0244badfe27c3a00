#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02t; mkdir -p $O
L="libfmmgpu_p0t0.so libfmmgpu_p0t1.so libfmmgpu_p1t0.so libfmmgpu_p1t1.so libfmmgpu_p2t1.so libfmmgpu_p0t0.so"
timeout 900 python tools/eval_ab.py FMMGPU_LIB $L > $O/ab_B.txt 2>&1
N=20000000 H=8 DIST=ellipsoid timeout 1200 python tools/eval_ab.py FMMGPU_LIB $L > $O/ab_D.txt 2>&1
cat $O/ab_*.txt
