mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 200 -k "pipelined or deterministic or run_entry" > gpurun_out/pytest_pipe.log 2>&1
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
