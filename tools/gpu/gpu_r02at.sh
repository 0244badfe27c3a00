#!/bin/bash
# phase-A table lookups deferred behind the slice's DMMAs (libfmmgpu_pf.so) vs current
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02at; mkdir -p $O
{
timeout 600 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_pf.so libfmmgpu.so libfmmgpu_pf.so
ORDER=6 H=7 timeout 600 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_pf.so
for lib in libfmmgpu.so libfmmgpu_pf.so; do
  FMMGPU_LIB=$lib timeout 300 python tools/scratch/field_hash.py
  FMMGPU_LIB=$lib timeout 300 python tools/scratch/field_hash.py 2000000 8 5 ellipsoid
done
} > $O/ab.log 2>&1
grep -v Warn $O/ab.log
