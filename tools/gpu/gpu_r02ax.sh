#!/bin/bash
# near-field CTA size: 11 warps (164 registers) and 13 warps (128) vs 12 (164)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ax; mkdir -p $O
{
timeout 600 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_w11.so libfmmgpu_w13.so libfmmgpu.so libfmmgpu_w11.so libfmmgpu_w13.so
N=20000000 H=8 DIST=ellipsoid timeout 600 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_w11.so libfmmgpu_w13.so
} > $O/ab.log 2>&1
grep -v Warn $O/ab.log
