#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ag; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q > $O/pytest_cfg.log 2>&1; echo "exit $?" >> $O/pytest_cfg.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench_B.json 2> $O/bench_B.err
timeout 900 python bench.py --config C --no-cpu-baseline > $O/bench_C.json 2> $O/bench_C.err
timeout 900 python bench.py --config E --no-cpu-baseline > $O/bench_E.json 2> $O/bench_E.err
for f in $O/pytest.log $O/pytest_cfg.log; do tail -2 $f; done
for c in B C E; do python -c "import json; d=json.load(open('$O/bench_$c.json')); print('$c', d['ms_per_step'], d['tree_build_ms'], d['lists_build_ms'], d['e2e']['value'], d['per_operator']['P2P']['ms_isolated'], d['roofline']['frac'])"; done
