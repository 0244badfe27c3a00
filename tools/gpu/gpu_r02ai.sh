#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ai; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "tree or lists or config or deep or summary" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 1500 python bench.py --config E > $O/bench_E.json 2> $O/bench_E.err
timeout 900 python bench.py > $O/bench_B.json 2> $O/bench_B.err
tail -2 $O/pytest.log
for c in B E; do python -c "import json; d=json.load(open('$O/bench_$c.json')); print('$c', d['ms_per_step'], d['tree_build_ms'], d['lists_build_ms'], d['e2e']['value'])"; done
