#!/bin/bash
# phase A at l <= 5 with 128-row M-tiles (8 warps of 32 x 32, 16-wide slices) vs 64-row
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02au; mkdir -p $O
{
FMMGPU_LIB=libfmmgpu_pa.so timeout 600 python tools/eval_ab.py FMMGPU_PA128 0 1 0 1
FMMGPU_LIB=libfmmgpu_pa.so N=100000 H=4 timeout 600 python tools/eval_ab.py FMMGPU_PA128 0 1
FMMGPU_LIB=libfmmgpu_pa.so N=20000000 H=8 DIST=ellipsoid timeout 600 python tools/eval_ab.py FMMGPU_PA128 0 1
for v in 0 1; do
  FMMGPU_PA128=$v FMMGPU_LIB=libfmmgpu_pa.so timeout 300 python tools/scratch/field_hash.py
  FMMGPU_PA128=$v FMMGPU_LIB=libfmmgpu_pa.so timeout 300 python tools/scratch/field_hash.py 2000000 8 5 ellipsoid
done
} > $O/ab.log 2>&1
grep -v Warn $O/ab.log
