mkdir -p gpurun_out
timeout 600 python tools/m2l_variants.py > gpurun_out/m2l_variants.log 2>&1
