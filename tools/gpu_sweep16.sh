cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s16_build.log 2>&1
timeout 900 python -m pytest tests/test_hier_gpu.py tests/test_multirank_emulated_gpu.py -x -q > gpurun_out/s16_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s16_pytest.log
timeout 900 python tools/sweep_grid.py C5 "NC_TABLES_FILE=tables/exp/C5_r126.npz" "NC_TABLES_FILE=tables/exp/C5_r126_t10.npz" > gpurun_out/s16_sweep_c5.jsonl 2>&1
NC_TABLES_FILE=tables/exp/C3_r126_t10.npz timeout 600 python tools/tol_calibration.py C3 1000 > gpurun_out/s16_tol_c3.jsonl 2>gpurun_out/s16_tol.err
NC_TABLES_FILE=tables/exp/C3_r126.npz timeout 600 python tools/tol_calibration.py C3 1000 >> gpurun_out/s16_tol_c3.jsonl 2>>gpurun_out/s16_tol.err
echo done
