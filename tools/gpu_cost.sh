# grid-vs-near cost model re-sweep after the step-4 / transform speedups: C5 time per constant, C3/C4 error (GPU box)
cd $GRAFT_REPO_ROOT
T=${1:-cost}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python tools/sweep_grid.py C5 "NC_COST_INTERP=0.15" "NC_COST_INTERP=0.12" "NC_COST_INTERP=0.10" "NC_COST_TRANSFORM=0.08" "NC_COST_INTERP=0.12;NC_COST_TRANSFORM=0.08" > gpurun_out/${T}_sweep_c5.jsonl 2>&1
for v in 0.15 0.12 0.10; do
  for c in C3 C4; do
    NC_COST_INTERP=$v timeout 600 python tools/hier_accuracy.py $c 1e-9 | sed "s/^{/{\"cost_interp\": $v, /" >> gpurun_out/${T}_acc.jsonl 2>&1
  done
done
echo done
