#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ab; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_configs.py -k "C" -x -q > $O/pytest_cfg.log 2>&1; echo "exit $?" >> $O/pytest_cfg.log
timeout 900 python bench.py --config C --steps 10 --warmup 3 > $O/bench_C.json 2> $O/bench_C.err
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_m2l_phase_a2" -s 4 -c 1 -o $O/C_m2la -f python tools/profile_eval.py 10000000 7 7 1 > $O/C_m2la.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_m2l_phase_b" -s 5 -c 1 -o $O/C_m2lb -f python tools/profile_eval.py 10000000 7 7 1 > $O/C_m2lb.out 2>&1
for f in $O/pytest.log $O/pytest_cfg.log; do tail -2 $f; done; head -c 400 $O/bench_C.json
