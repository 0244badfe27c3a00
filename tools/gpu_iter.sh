mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python tools/eval_ab.py FMMGPU_P2P_VARIANT 0 > gpurun_out/eval_ab.log 2>&1
