# k_transform with paired (cos, sin) twiddle reads: C5/C4 timing + hierarchical GPU tests (GPU box)
cd $GRAFT_REPO_ROOT
T=${1:-tr}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 600 python tools/sweep_grid.py C5 "NC_INTERP_VARIANT=128,2,3,4" "NC_INTERP_VARIANT=128,2,3,4" > gpurun_out/${T}_sweep_c5.jsonl 2>&1
timeout 600 python tools/sweep_grid.py C4 "NC_INTERP_VARIANT=128,2,3,4" > gpurun_out/${T}_sweep_c4.jsonl 2>&1
timeout 900 python -m pytest tests/test_hier_gpu.py -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
CMD="python bench.py --steps 1 --warmup 1 --no-solve --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_launch.log 2>&1
echo done
