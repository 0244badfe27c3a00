#!/bin/bash
# round-2 first GPU pass: gpu tests (config parity evidence), default bench, reference arm
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02a
nproc > gpurun_out/r02a/nproc.txt; lscpu > gpurun_out/r02a/lscpu.txt; free -g >> gpurun_out/r02a/lscpu.txt
nvidia-smi > gpurun_out/r02a/smi.txt
FMMGPU_PARITY_OUT=gpurun_out/r02a timeout 2400 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r02a/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02a/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02a/bench.json 2> gpurun_out/r02a/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r02a/bench_ref.json 2> gpurun_out/r02a/bench_ref.err
tail -3 gpurun_out/r02a/pytest_gpu.log; cat gpurun_out/r02a/bench.json gpurun_out/r02a/bench_ref.json
