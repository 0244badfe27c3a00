# A/B of a launch switch at config B (development aid)
mkdir -p gpurun_out
{
timeout 600 python tools/op_variants.py FMMGPU_STAGE_SERIAL P2P 7 0 1
timeout 600 python tools/eval_ab.py FMMGPU_STAGE_SERIAL 0 1 0 1
} > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log | grep -v Warn
