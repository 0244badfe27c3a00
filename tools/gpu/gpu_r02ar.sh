#!/bin/bash
# co-residency with a common (max shared) carveout: P2P CTA size x CTAs per SM
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ar; mkdir -p $O
{
for lib in libfmmgpu.so libfmmgpu_w8.so libfmmgpu_w6.so; do
  echo "== $lib carve"
  FMMGPU_CARVE=1 FMMGPU_LIB=$lib timeout 600 python tools/eval_ab.py FMMGPU_MU_CPS 0 1
done
for lib in libfmmgpu_w8.so libfmmgpu_w6.so; do
  echo "== $lib C carve"
  FMMGPU_CARVE=1 ORDER=7 FMMGPU_LIB=$lib timeout 600 python tools/eval_ab.py FMMGPU_MU_CPS 1
done
} > $O/ab.log 2>&1
grep -v Warn $O/ab.log
