cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s15_build.log 2>&1
timeout 900 python tools/sweep_grid.py C5 "NC_TABLES_FILE=tables/exp/C5_r1414.npz" "NC_TABLES_FILE=tables/exp/C5_r126.npz" > gpurun_out/s15_sweep_c5.jsonl 2>&1
NC_TABLES_FILE=tables/exp/C3_r126.npz timeout 600 python tools/tol_calibration.py C3 1000 > gpurun_out/s15_tol_c3.jsonl 2>gpurun_out/s15_tol.err
echo done
