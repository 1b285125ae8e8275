cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s2_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s2_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s2_pytest_gpu.log
timeout 1200 python tools/sweep_grid.py C5 "2,4,0,256,0" "2,2,0,256,1" "2,4,0,256,1" "2,1,0,256,1" "4,2,0,256,1" "2,4,0,128,1" "2,4,0,512,1" > gpurun_out/s2_sweep_c5.jsonl 2>&1
for c in C3 C4; do
timeout 600 python tools/tol_calibration.py $c 300 1000 3000 10000 >> gpurun_out/s2_tol.jsonl 2>>gpurun_out/s2_tol.err
NC_GRID_VARIANT=2,4,0,256,1 timeout 600 python tools/tol_calibration.py $c 300 1000 3000 10000 >> gpurun_out/s2_tol.jsonl 2>>gpurun_out/s2_tol.err
done
NC_GRID_VARIANT=2,4,0,256,1 timeout 600 python tools/tol_calibration.py C5 300 1000 3000 >> gpurun_out/s2_tol.jsonl 2>>gpurun_out/s2_tol.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err
echo done
