#!/bin/bash
# auto P2P kernel choice: full GPU suite, config A bench line, tree/e2e trace probe
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02j; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q -rs > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py --config A --steps 10 --warmup 3 > $O/bench_A.json 2> $O/bench_A.err
FMMGPU_TRACE=1 timeout 300 python tools/scratch/e2e_probe.py > $O/e2e_probe.txt 2>&1
tail -3 $O/pytest_gpu.log; head -c 400 $O/bench_A.json
