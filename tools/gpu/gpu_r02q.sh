#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02q; mkdir -p $O
ORDER=7 timeout 900 python tools/eval_ab.py FMMGPU_M2L_MS_MIN 1 2 4 8 > $O/ab_msmin_C.txt 2>&1
timeout 600 python tools/eval_ab.py FMMGPU_M2L_MS_MIN 1 2 4 > $O/ab_msmin_B.txt 2>&1
cat $O/*.txt
