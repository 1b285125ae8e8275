cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s7_build.log 2>&1
timeout 600 python -m pytest tests/test_hier_gpu.py -x -q -k "C2 or far" > gpurun_out/s7_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s7_pytest.log
timeout 1500 python tools/sweep_grid.py C5 "NC_INTERP_VARIANT=128,4,1" "NC_INTERP_VARIANT=128,4,2" "NC_INTERP_VARIANT=256,2,4" "NC_INTERP_VARIANT=256,2,2" "NC_INTERP_VARIANT=256,1,4" "NC_INTERP_VARIANT=256,1,8" "NC_INTERP_VARIANT=128,2,4" > gpurun_out/s7_sweep_interp.jsonl 2>&1
timeout 1500 python tools/sweep_grid.py C5 "NC_COST_NEAR=1.0" "NC_COST_NEAR=1.4" "NC_COST_NEAR=1.4;NC_COST_INTERP=0.15" "NC_COST_NEAR=1.0;NC_COST_INTERP=0.15" "NC_COST_NEAR=0.8" "NC_COST_INTERP=0.03" > gpurun_out/s7_sweep_cost.jsonl 2>&1
echo done
