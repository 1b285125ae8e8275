# step-4 interpolation variants (k_interp MB=0: angular sums first, j accumulators in registers) on C5 (GPU box)
cd $GRAFT_REPO_ROOT
T=${1:-ip}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 1200 python tools/sweep_grid.py C5 "NC_INTERP_VARIANT=128,4,1,4" "NC_INTERP_VARIANT=256,2,0,2" "NC_INTERP_VARIANT=256,2,0,3" \
  "NC_INTERP_VARIANT=128,4,0,4" "NC_INTERP_VARIANT=128,2,0,6" > gpurun_out/${T}_sweep_c5.jsonl 2>&1
for v in "128,4,1,4" "256,2,0,2"; do
  for c in C3 C4; do
    NC_INTERP_VARIANT=$v timeout 600 python tools/hier_accuracy.py $c 1e-9 | sed "s/^{/{\"interp\": \"$v\", /" >> gpurun_out/${T}_acc.jsonl 2>&1
  done
done
M=smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,local_load_bytes,l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum
for v in "128,4,1,4" "256,2,0,2"; do
  NC_INTERP_VARIANT=$v timeout 600 ncu --metrics $M --clock-control none -k regex:k_interp -c 1 --csv python tools/hier_probe.py C4 > gpurun_out/${T}_ncu_${v//,/_}.csv 2>&1
done
echo done
