#!/bin/bash
# round-2 closing evidence on the final kernels: GPU tests, smoke, bench lines A-E with
# same-config reference baselines and parity, the reference arm, launch list + ncu of the
# top kernels at B, scaling projection
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/final5; mkdir -p $O
nproc > $O/host.txt; free -g >> $O/host.txt; nvidia-smi >> $O/host.txt
timeout 1800 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_B.json 2> $O/bench_B.err
timeout 900 python bench.py --impl reference > $O/bench_reference_B.json 2> $O/bench_reference_B.err
for cfg in A C D E; do
  timeout 1500 python bench.py --config $cfg --steps 10 --warmup 3 > $O/bench_$cfg.json 2> $O/bench_$cfg.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_|Radix|Scan|RunLength|Reduce" --csv --log-file $O/launches.csv python tools/profile_eval.py 10000000 7 5 2 > $O/launches.out 2>&1
cap() {
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$2" -s "$3" -c 1 -o $O/$1 -f python tools/profile_eval.py 10000000 7 5 1 > $O/$1.out 2>&1
}
cap prof_p2p 'k_p2p_mutual' 0
cap prof_l2p "k_l2p_block" 0
cap prof_m2la 'k_m2l_phase_a' 4
cap prof_m2lb 'k_m2l_phase_b' 4
timeout 900 python tools/scaling_projection.py B > $O/scaling_projection_B.json 2> $O/scaling.err
tail -3 $O/pytest_gpu.log; tail -1 $O/smoke.log; for f in $O/bench_*.json; do echo $f; head -c 200 $f; echo; done
