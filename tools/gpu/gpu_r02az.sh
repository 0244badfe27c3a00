#!/bin/bash
# phase-A epilogue: targets read before the scatter stores (libfmmgpu_ep.so) vs current
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02az; mkdir -p $O
{
timeout 600 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_ep.so libfmmgpu.so libfmmgpu_ep.so
for lib in libfmmgpu.so libfmmgpu_ep.so; do
  FMMGPU_LIB=$lib timeout 300 python tools/scratch/field_hash.py
  FMMGPU_LIB=$lib timeout 300 python tools/scratch/field_hash.py 2000000 8 5 ellipsoid
done
} > $O/ab.log 2>&1
grep -v Warn $O/ab.log
