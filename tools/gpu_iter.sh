mkdir -p gpurun_out
FMMGPU_TRACE=1 PROBE_CFG=D timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe_D.log 2>&1
timeout 900 python bench.py --config D --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_D.json 2> gpurun_out/bench_D.err
