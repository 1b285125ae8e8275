cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s10_build.log 2>&1
timeout 900 python -m pytest tests/test_hier_gpu.py -x -q -k "C2 or C3 or far" > gpurun_out/s10_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s10_pytest.log
for c in C5; do NC_HIER_DIAG=1 timeout 300 python tools/hier_probe.py $c > gpurun_out/s10_diag_$c.log 2>&1; done
timeout 900 python tools/sweep_grid.py C5 "NC_MAX_GRIDS=2" "NC_MAX_GRIDS=3" "NC_MAX_GRIDS=3;NC_COST_INTERP=0.15" > gpurun_out/s10_sweep_c5.jsonl 2>&1
for c in C3 C5; do timeout 600 python tools/tol_calibration.py $c 1000 >> gpurun_out/s10_tol.jsonl 2>>gpurun_out/s10_tol.err; done
echo done
