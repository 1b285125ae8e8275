cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s6_build.log 2>&1
timeout 900 python -m pytest tests/test_hier_gpu.py tests/test_multirank_emulated_gpu.py -x -q > gpurun_out/s6_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s6_pytest.log
timeout 1200 python tools/sweep_grid.py C5 "128,2,4,256,0,0,8" "128,2,4,256,1,0,8" "128,2,4,256,1,0,4" "256,1,4,256,1,0,6" > gpurun_out/s6_sweep_c5.jsonl 2>&1
echo done
