mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "coincident or edge or tree" 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_leaf_scan --csv python tools/profile_eval.py 10000000 7 5 0 2>&1 | grep leaf_scan | tail -1 | awk -F, '{print $NF}'
