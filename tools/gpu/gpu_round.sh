#!/bin/bash
# One GPU session: parity tests, smoke, ncu launch list and full capture of the top kernels.
# usage: tools/gpu_round.sh [tests] [quick] [launches] [full] [bench]   (FULL_RE / FULL_SKIP / FULL_COUNT)
mkdir -p gpurun_out
for what in "$@"; do
case "$what" in
  tests) timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
         timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1 ;;
  launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_|Radix|Scan|RunLength|Reduce" --csv --log-file gpurun_out/launches.csv python tools/profile_eval.py 10000000 7 5 2 > gpurun_out/launches.out 2>&1 ;;
  full) timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$FULL_RE" -s "${FULL_SKIP:-0}" -c "${FULL_COUNT:-1}" -o gpurun_out/prof -f python tools/profile_eval.py 10000000 7 5 1 > gpurun_out/prof.out 2>&1 ;;
  full2) timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$FULL2_RE" -s "${FULL2_SKIP:-0}" -c "${FULL2_COUNT:-1}" -o gpurun_out/prof2 -f python tools/profile_eval.py 10000000 7 5 1 > gpurun_out/prof2.out 2>&1 ;;
  quick) timeout 300 python tools/quick_eval.py > gpurun_out/quick.log 2>&1 ;;
  bench) timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err ;;
esac
done
# configs: every BASELINE.json config through bench.py (short runs)
if [ "${ALLCONFIGS:-0}" = "1" ]; then
  for cfgname in A B C D E; do
    timeout 900 python bench.py --config $cfgname --steps 5 --warmup 3 > gpurun_out/bench_$cfgname.json 2> gpurun_out/bench_$cfgname.err
  done
fi
