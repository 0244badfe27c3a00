#!/bin/bash
# near-field stream entries located by a forward segment cursor (libfmmgpu_cur.so) vs binary search
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ay; mkdir -p $O
{
timeout 600 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_cur.so libfmmgpu.so libfmmgpu_cur.so
N=20000000 H=8 DIST=ellipsoid timeout 600 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_cur.so
N=100000000 H=8 timeout 900 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_cur.so
for lib in libfmmgpu.so libfmmgpu_cur.so; do
  FMMGPU_LIB=$lib timeout 300 python tools/scratch/field_hash.py
  FMMGPU_LIB=$lib timeout 300 python tools/scratch/field_hash.py 2000000 8 5 ellipsoid
done
} > $O/ab.log 2>&1
grep -v Warn $O/ab.log
