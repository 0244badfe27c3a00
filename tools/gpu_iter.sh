mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
ORDER=7 timeout 900 python tools/eval_ab.py FMMGPU_X 0 > gpurun_out/eval_ab.log 2>&1
