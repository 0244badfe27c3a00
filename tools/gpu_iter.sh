mkdir -p gpurun_out
ORDER=7 timeout 900 python tools/eval_ab.py FMMGPU_M2L_A7 0 1 > gpurun_out/eval_ab.log 2>&1
