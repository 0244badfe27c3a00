#!/bin/bash
# L2P (fused slot drain) at 5 / 6 CTAs per SM (96 / 80 registers, small spills) vs 4
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02be; mkdir -p $O
{
timeout 600 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_l5.so libfmmgpu_l6.so libfmmgpu.so libfmmgpu_l5.so libfmmgpu_l6.so
N=100000000 H=8 timeout 900 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_l5.so libfmmgpu_l6.so
for lib in libfmmgpu.so libfmmgpu_l5.so libfmmgpu_l6.so; do
  FMMGPU_LIB=$lib timeout 300 python tools/scratch/field_hash.py
done
} > $O/ab.log 2>&1
grep -v Warn $O/ab.log
