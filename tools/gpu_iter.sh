mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
FMMGPU_TRACE=1 timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
