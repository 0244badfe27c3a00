#!/bin/bash
# phase B: Yt row pointers resolved once per CTA (libfmmgpu_pb.so, includes the phase-A epilogue change) vs ep only
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ba; mkdir -p $O
{
timeout 600 python tools/eval_ab.py FMMGPU_LIB libfmmgpu_ep.so libfmmgpu_pb.so libfmmgpu_ep.so libfmmgpu_pb.so
ORDER=7 timeout 600 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_ep.so libfmmgpu_pb.so
for lib in libfmmgpu.so libfmmgpu_pb.so; do
  FMMGPU_LIB=$lib timeout 300 python tools/scratch/field_hash.py
  FMMGPU_LIB=$lib timeout 300 python tools/scratch/field_hash.py 2000000 8 5 ellipsoid
  FMMGPU_LIB=$lib timeout 300 python tools/scratch/field_hash.py 1000000 6 7 uniform
done
} > $O/ab.log 2>&1
grep -v Warn $O/ab.log
