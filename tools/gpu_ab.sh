# A/B of a launch switch at config B (development aid)
mkdir -p gpurun_out
{
timeout 600 python tools/op_variants.py FMMGPU_NONE L2P 7 0
ORDER=7 timeout 600 python tools/op_variants.py FMMGPU_NONE L2P 7 0
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "operators or full_evaluation" 2>&1 | tail -2
} > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log | grep -v Warn
