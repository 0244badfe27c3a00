mkdir -p gpurun_out
timeout 600 python tools/p2p_variants.py > gpurun_out/p2p_variants.log 2>&1
