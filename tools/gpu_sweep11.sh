cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s11_build.log 2>&1
timeout 900 python tools/sweep_grid.py C5 "NC_INTERP_VARIANT=128,4,1" "NC_INTERP_VARIANT=0,0,0" "NC_MAX_GRIDS=2" > gpurun_out/s11_sweep_c5.jsonl 2>&1
timeout 900 python tools/sweep_grid.py C4 "NC_INTERP_VARIANT=128,4,1" "NC_INTERP_VARIANT=0,0,0" > gpurun_out/s11_sweep_c4.jsonl 2>&1
timeout 900 python -m pytest tests/test_hier_gpu.py tests/test_multirank_emulated_gpu.py -x -q > gpurun_out/s11_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s11_pytest.log
echo done
