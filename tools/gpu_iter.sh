mkdir -p gpurun_out
timeout 600 python tools/eval_ab.py FMMGPU_M2L_WAVES 1 2 4 1 > gpurun_out/eval_ab.log 2>&1
