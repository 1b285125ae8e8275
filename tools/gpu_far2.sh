# far-table variants round 2: C5 timing sweep + shared-memory wavefront counts per variant (ncu, C4, one launch)
cd $GRAFT_REPO_ROOT
T=${1:-far2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python tools/sweep_grid.py C5 "128,2,4,256,2,0,6" "128,2,4,256,5,0,8" "128,2,4,256,5,0,6" "128,2,4,256,6,0,8" \
  "128,2,2,256,5,0,8" "256,1,4,256,5,0,4" "128,2,4,256,1" > gpurun_out/${T}_sweep_c5.jsonl 2>&1
M=l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed
for v in "128,2,4,256,1" "128,2,4,256,2,0,6" "128,2,4,256,5,0,8" "128,2,4,256,6,0,8"; do
  NC_GRID_VARIANT=$v timeout 600 ncu --metrics $M --clock-control none -k regex:k_pairs_grid -c 1 --csv python tools/hier_probe.py C4 > gpurun_out/${T}_ncu_${v//,/_}.csv 2>&1
done
echo done
