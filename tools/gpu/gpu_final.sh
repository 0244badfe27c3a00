#!/bin/bash
# Round evidence in one GPU session: parity tests, smoke, launch list and ncu --set full
# of the top kernels of one config-B evaluation (-> gpurun_out/final/), and every
# BASELINE.json config through bench.py plus the reference arm at config B.
set -u
mkdir -p gpurun_out/final
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/final/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_|Radix|Scan|RunLength|Reduce" \
  --csv --log-file gpurun_out/final/launches.csv python tools/profile_eval.py 10000000 7 5 2 > gpurun_out/final/launches.out 2>&1
cap() {  # tag regex skip
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" -s "$3" -c 1 \
    -o "gpurun_out/final/prof_$1" -f python tools/profile_eval.py 10000000 7 5 1 > "gpurun_out/final/prof_$1.out" 2>&1
}
cap p2p 'k_p2p' 0
cap m2la 'k_m2l_phase_a' 4
cap m2lb 'k_m2l_phase_b' 4
cap p2m 'k_p2m' 0
cap l2p 'k_l2p' 0
cap gather 'k_gather' 0
cap m2m 'k_transfer_warp' 0
for cfgname in A B C D E; do
  timeout 900 python bench.py --config $cfgname --steps 5 --warmup 3 > gpurun_out/final/bench_$cfgname.json 2> gpurun_out/final/bench_$cfgname.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final/bench_ref_B.json 2> gpurun_out/final/bench_ref_B.err
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
