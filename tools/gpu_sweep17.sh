cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s17_build.log 2>&1
timeout 900 python -m pytest tests/test_hier_gpu.py -x -q -k "C2 or C3" > gpurun_out/s17_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s17_pytest.log
T=tables/exp/C5_r126_t10.npz
timeout 1200 python tools/sweep_grid.py C5 "NC_TABLES_FILE=$T" "NC_TABLES_FILE=$T;NC_GRID_VARIANT=256,1,4,256,1,0,6" "NC_TABLES_FILE=$T;NC_GRID_VARIANT=256,2,2,256,1,0,5" "NC_TABLES_FILE=$T;NC_GRID_VARIANT=256,1,4,256,1,0,5" > gpurun_out/s17_sweep_c5.jsonl 2>&1
NC_TABLES_FILE=tables/exp/C3_r126_t10.npz timeout 600 python tools/tol_calibration.py C3 1000 > gpurun_out/s17_tol_c3.jsonl 2>gpurun_out/s17_tol.err
echo done
