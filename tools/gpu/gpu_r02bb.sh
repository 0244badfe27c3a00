#!/bin/bash
# streamed phase A (l >= 6) epilogue: targets read before the stores (libfmmgpu_a2.so) vs current
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bb; mkdir -p $O
{
ORDER=7 timeout 600 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_a2.so libfmmgpu.so libfmmgpu_a2.so
ORDER=6 timeout 600 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_a2.so
for lib in libfmmgpu.so libfmmgpu_a2.so; do
  FMMGPU_LIB=$lib timeout 300 python tools/scratch/field_hash.py 1000000 6 7 uniform
  FMMGPU_LIB=$lib timeout 300 python tools/scratch/field_hash.py 2000000 7 6 ellipsoid
done
} > $O/ab.log 2>&1
grep -v Warn $O/ab.log
