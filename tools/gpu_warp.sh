# warp-level grid-kernel work units (tma = 3) vs the CTA-unit kernel on C5 and C4 (GPU box)
cd $GRAFT_REPO_ROOT
T=${1:-wp}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 1500 python tools/sweep_grid.py C5 "128,2,4,256,5,0,8" "8,2,4,64,5,3,4" "8,2,4,96,5,3,4" "4,2,4,64,5,3,8" "8,2,2,64,5,3,4" \
  "8,2,4,64,5,3,3" "8,2,4,32,5,3,4" > gpurun_out/${T}_sweep_c5.jsonl 2>&1
timeout 600 python tools/sweep_grid.py C4 "128,2,4,256,5,0,8" "8,2,4,64,5,3,4" > gpurun_out/${T}_sweep_c4.jsonl 2>&1
M=smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio
NC_GRID_VARIANT="8,2,4,64,5,3,4" timeout 600 ncu --metrics $M --clock-control none -k regex:k_pairs_grid -c 1 --csv python tools/hier_probe.py C4 > gpurun_out/${T}_ncu_w.csv 2>&1
echo done
