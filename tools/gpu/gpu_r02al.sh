#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02al; mkdir -p $O
timeout 1200 python -m pytest tests/test_multigpu.py tests/test_dist_input.py -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 900 python tools/scaling_projection.py B > $O/scaling_projection_B.json 2> $O/scaling.err
tail -2 $O/pytest.log; python -c "
import json; d=json.load(open('$O/scaling_projection_B.json'))
for r in d['rows']: print(r['gpus'], round(r['max_rank_ms'],3), round(r['projected_ms'],3), round(r['efficiency'],3))"
