# direct mode with the exact-form table (green_exact_r) vs the mantissa table: parity tests + C2 direct bench (GPU box)
cd $GRAFT_REPO_ROOT
T=${1:-dx}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python -m pytest tests/test_direct_gpu.py tests/test_hier_gpu.py tests/test_multirank_emulated_gpu.py -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 600 python bench.py --config C2 --mode direct --no-cpu-baseline > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
NC_EXACT_TABLE=0 timeout 600 python bench.py --config C2 --mode direct --no-cpu-baseline --no-solve > gpurun_out/${T}_bench_c2_old.json 2>> gpurun_out/${T}_bench_c2.err
M=smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed
timeout 600 ncu --metrics $M --clock-control none -k regex:k_pairs_direct -c 1 --csv python bench.py --config C2 --mode direct --no-cpu-baseline --no-solve --steps 1 --warmup 1 > gpurun_out/${T}_ncu_new.csv 2>&1
NC_EXACT_TABLE=0 timeout 600 ncu --metrics $M --clock-control none -k regex:k_pairs_direct -c 1 --csv python bench.py --config C2 --mode direct --no-cpu-baseline --no-solve --steps 1 --warmup 1 > gpurun_out/${T}_ncu_old.csv 2>&1
echo done
