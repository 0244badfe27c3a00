# ncu --set full of the leaf-level M2L phases at config C (order 7)
mkdir -p gpurun_out
for k in a b; do
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_m2l_phase_$k" -s 4 -c 1 \
  -o gpurun_out/prof_c_m2l$k -f python tools/profile_eval.py 10000000 7 7 1 > gpurun_out/prof_c_m2l$k.out 2>&1
done
ls -la gpurun_out/prof_c_*
