#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02x; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_dist_input.py -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_configs.py -k "B or D" -x -q > $O/pytest_cfg.log 2>&1; echo "exit $?" >> $O/pytest_cfg.log
FMMGPU_TRACE=1 timeout 300 python tools/scratch/e2e_probe.py > $O/e2e_probe.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
for f in $O/pytest.log $O/pytest_cfg.log; do tail -2 $f; done; grep -v "alloc\]\|\[tree\]\|readback\|pipe\]" $O/e2e_probe.txt; head -c 300 $O/bench.json
