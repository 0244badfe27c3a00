#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ad; mkdir -p $O
N=20000000 H=8 DIST=ellipsoid timeout 1200 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_t192.so libfmmgpu_t256.so > $O/ab_D.txt 2>&1
cat $O/ab_D.txt
