#!/bin/bash
# re-entry check of the committed tree: GPU tests, smoke, bench B (device + e2e + parity)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${OUT:-r02ap}; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_B.json 2> $O/bench_B.err
tail -3 $O/pytest_gpu.log; tail -1 $O/smoke.log; head -c 400 $O/bench_B.json
