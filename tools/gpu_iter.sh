mkdir -p gpurun_out
timeout 900 python tools/eval_ab.py FMMGPU_PRIO 0 1 2 0 > gpurun_out/eval_ab.log 2>&1
