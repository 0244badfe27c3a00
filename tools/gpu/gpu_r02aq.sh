#!/bin/bash
# co-residency of the near-field kernel with the far chain: P2P CTA size x CTAs per SM
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02aq; mkdir -p $O
{
for lib in libfmmgpu.so libfmmgpu_w8.so libfmmgpu_w6.so libfmmgpu_w4.so; do
  echo "== $lib"
  FMMGPU_LIB=$lib timeout 600 python tools/eval_ab.py FMMGPU_MU_CPS 0 1 2
done
echo "== config C"
for lib in libfmmgpu.so libfmmgpu_w8.so libfmmgpu_w6.so; do
  echo "== $lib C"
  ORDER=7 FMMGPU_LIB=$lib timeout 600 python tools/eval_ab.py FMMGPU_MU_CPS 0 1
done
} > $O/ab.log 2>&1
grep -v Warn $O/ab.log
