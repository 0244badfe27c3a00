mkdir -p gpurun_out
FMMGPU_TRACE=1 timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "pipelined" > gpurun_out/pytest_pipe.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
