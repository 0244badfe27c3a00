#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02o; mkdir -p $O
timeout 900 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_pa1.so libfmmgpu_pa2.so libfmmgpu_pa3.so > $O/ab_B.txt 2>&1
ORDER=7 timeout 900 python tools/eval_ab.py FMMGPU_LIB libfmmgpu.so libfmmgpu_pa4.so > $O/ab_C.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -k deep -q -rs -s > $O/pytest_deep.log 2>&1; echo "exit $?" >> $O/pytest_deep.log
cat $O/ab_*.txt; grep "deep tree" $O/pytest_deep.log; tail -1 $O/pytest_deep.log
