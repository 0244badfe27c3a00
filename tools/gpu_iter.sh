mkdir -p gpurun_out
timeout 900 python tools/scaling_projection.py B > gpurun_out/scaling_B.json 2> gpurun_out/scaling_B.err
timeout 1800 python tools/scaling_projection.py E > gpurun_out/scaling_E.json 2> gpurun_out/scaling_E.err
