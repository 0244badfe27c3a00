#!/bin/bash
# near field: target position loaded a ring step ahead (libfmmgpu_pt.so) vs current
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bf; mkdir -p $O
{
timeout 600 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_pt.so libfmmgpu.so libfmmgpu_pt.so
N=20000000 H=8 DIST=ellipsoid timeout 600 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_pt.so
for lib in libfmmgpu.so libfmmgpu_pt.so; do
  FMMGPU_LIB=$lib timeout 300 python tools/scratch/field_hash.py
  FMMGPU_LIB=$lib timeout 300 python tools/scratch/field_hash.py 2000000 8 5 ellipsoid
done
} > $O/ab.log 2>&1
grep -v Warn $O/ab.log
