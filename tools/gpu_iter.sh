mkdir -p gpurun_out
timeout 600 python tools/p2p_variants.py > gpurun_out/p2p_variants.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "p2p or full_evaluation or determin" > gpurun_out/pytest_p2p.log 2>&1
