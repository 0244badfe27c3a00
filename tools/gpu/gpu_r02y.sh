#!/bin/bash
# executed FP64 operations per kernel of one config-B evaluation (ncu instruction counters)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02y; mkdir -p $O
M=sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,gpu__time_duration.sum
timeout 900 ncu --metrics $M --clock-control none -k "regex:k_p2m|k_l2p|k_transfer|k_p2p|k_m2l_phase|k_gather" --csv --log-file $O/fp64_ops.csv python tools/profile_eval.py 10000000 7 5 1 > $O/fp64_ops.out 2>&1
head -5 $O/fp64_ops.csv; tail -3 $O/fp64_ops.out
