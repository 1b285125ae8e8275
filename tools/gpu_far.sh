# far-table grid-kernel variants (R25): C5/C4 timing sweep + C3/C4 hier-vs-direct error per variant (GPU box)
cd $GRAFT_REPO_ROOT
T=${1:-far}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python tools/sweep_grid.py C5 "128,2,4,256,1" "128,2,4,256,2" "128,2,4,256,3" "128,2,4,256,4" \
  "128,2,4,256,2,0,6" "256,2,2,256,2,0,3" "128,2,4,512,2" > gpurun_out/${T}_sweep_c5.jsonl 2>&1
timeout 600 python tools/sweep_grid.py C4 "128,2,4,256,1" "128,2,4,256,2" "128,2,4,256,4" > gpurun_out/${T}_sweep_c4.jsonl 2>&1
for v in "128,2,4,256,0" "128,2,4,256,1" "128,2,4,256,2" "128,2,4,256,3" "128,2,4,256,4"; do
  for c in C3 C4; do
    NC_GRID_VARIANT=$v timeout 600 python tools/hier_accuracy.py $c 1e-9 | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/${T}_acc.jsonl 2>&1
  done
done
echo done
