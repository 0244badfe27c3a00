mkdir -p gpurun_out
timeout 900 python tools/eval_ab.py FMMGPU_M2L_PERSIST 0 1 2 0 1 > gpurun_out/eval_ab.log 2>&1
timeout 600 python tools/op_variants.py FMMGPU_M2L_PERSIST M2L 6 0 1 > gpurun_out/op.log 2>&1
