#!/bin/bash
# P2P register/occupancy variants (A/B): config B and D evaluations per library build
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02g; mkdir -p $O
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/mc tools/microbench/p2p_mutual_ceiling.cu && timeout 120 /tmp/mc > $O/mutual_ceiling.txt 2>&1
for cfg in B D; do
  if [ $cfg = D ]; then export N=20000000 H=8 DIST=ellipsoid; else unset N H DIST; fi
  timeout 900 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_w12.so libfmmgpu_w12ilv.so libfmmgpu_w8r255.so libfmmgpu_w12ts6.so libfmmgpu_w8ts6.so libfmmgpu_w10.so > $O/ab_$cfg.txt 2>&1
done
cat $O/*.txt
