# Shared-memory bank conflicts and pipe use of every kernel of one config-B evaluation
# (development aid) + whole-evaluation device time of the current build.
mkdir -p gpurun_out
: # eval timing skipped
timeout 900 ncu --clock-control none -k regex:^k_ --csv --log-file gpurun_out/bank.csv --metrics \
gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active \
  python tools/profile_eval.py 10000000 7 5 1 > gpurun_out/bank.out 2>&1
cat gpurun_out/eval.log
