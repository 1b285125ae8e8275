cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s1_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s1_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s1_pytest_gpu.log
timeout 1200 python tools/sweep_grid.py C5 "2,2,0,512" "2,2,0,256" "2,2,0,128" "2,1,0,256" "2,4,0,256" "2,2,1,512" "2,2,1,256" "2,2,1,128" "2,1,1,128" "2,4,1,256" "4,1,0,256" "4,2,0,256" "4,1,1,256" "4,2,1,256" "4,2,1,128" > gpurun_out/s1_sweep_c5.jsonl 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s1_bench.json 2> gpurun_out/s1_bench.err
echo done
