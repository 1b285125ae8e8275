# async (cp.async double-buffered) grid-kernel staging + separable step-4 for single-member groups (GPU box)
cd $GRAFT_REPO_ROOT
T=${1:-as}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
NC_HIER_DIAG=1 timeout 600 python tools/hier_probe.py C5 > gpurun_out/${T}_diag_c5.log 2>&1
timeout 1200 python tools/sweep_grid.py C5 "128,2,4,256,5,0,8;NC_INTERP_SEP=0" "128,2,4,256,5,0,8" "128,2,4,176,5,2,8" \
  "128,2,4,176,5,2,7" "128,2,4,256,5,2,7" "128,2,2,176,5,2,8" > gpurun_out/${T}_sweep_c5.jsonl 2>&1
for c in C3 C4; do
  NC_INTERP_SEP=0 timeout 600 python tools/hier_accuracy.py $c 1e-9 | sed "s/^{/{\"sep\": 0, /" >> gpurun_out/${T}_acc.jsonl 2>&1
  timeout 600 python tools/hier_accuracy.py $c 1e-9 | sed "s/^{/{\"sep\": 1, /" >> gpurun_out/${T}_acc.jsonl 2>&1
done
timeout 900 python -m pytest tests/test_hier_gpu.py -x -q > gpurun_out/${T}_pytest_hier.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_hier.log
echo done
