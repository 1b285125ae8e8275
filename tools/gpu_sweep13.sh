cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s13_build.log 2>&1
NC_HIER_DIAG=1 timeout 300 python tools/hier_probe.py C5 > gpurun_out/s13_diag_C5_base.log 2>&1
NC_HIER_DIAG=1 NC_TABLES_FILE=tables/exp/C5_r1414.npz timeout 300 python tools/hier_probe.py C5 > gpurun_out/s13_diag_C5_r1414.log 2>&1
timeout 900 python tools/sweep_grid.py C5 "NC_MAX_GRIDS=3" "NC_TABLES_FILE=tables/exp/C5_r1414.npz" > gpurun_out/s13_sweep_c5.jsonl 2>&1
NC_TABLES_FILE=tables/exp/C3_r1414.npz timeout 600 python tools/tol_calibration.py C3 1000 > gpurun_out/s13_tol_c3.jsonl 2>gpurun_out/s13_tol.err
timeout 600 python tools/tol_calibration.py C3 1000 >> gpurun_out/s13_tol_c3.jsonl 2>>gpurun_out/s13_tol.err
echo done
