# grid tolerance factor (R21) trade: hier-vs-direct error at C3/C4 and C5 time per factor (GPU box)
cd $GRAFT_REPO_ROOT
T=${1:-tol}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for f in 1000 1500 2000 3000; do
  for c in C3 C4; do
    NC_GRID_TOL_FACTOR=$f timeout 600 python tools/hier_accuracy.py $c 1e-9 >> gpurun_out/${T}_acc.jsonl 2>&1
  done
done
timeout 1200 python tools/sweep_grid.py C5 "NC_GRID_TOL_FACTOR=1000" "NC_GRID_TOL_FACTOR=1500" "NC_GRID_TOL_FACTOR=2000" "NC_GRID_TOL_FACTOR=3000" > gpurun_out/${T}_sweep_c5.jsonl 2>&1
echo done
