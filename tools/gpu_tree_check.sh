mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tree or edge or deterministic or pipelined" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_leaf_scan --csv python tools/profile_eval.py 10000000 7 5 0 2>&1 | grep leaf_scan | tail -2
timeout 600 python tools/pipe_trace.py > gpurun_out/pipe_trace.log 2>&1; grep -v Warn gpurun_out/pipe_trace.log | tail -60
