# A/B of a launch switch at config B (development aid)
mkdir -p gpurun_out
{
timeout 600 python tools/op_variants.py FMMGPU_P2P_VARIANT P2P 7 0 2 3
} > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log | grep -v Warn
