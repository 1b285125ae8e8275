# grid-size knob sweep, one process per setting (R21); usage (under gpurun): bash tools/gpu_margin_sweep.sh <tag> "<K=V,K=V> <K=V> ..."
cd $GRAFT_REPO_ROOT
T=$1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
O=gpurun_out/${T}_margin_sweep.jsonl; : > $O
NC_TUNING=1 NC_GRID_TOL_FACTOR=100 timeout 600 python tools/margin_sweep.py ref 2> gpurun_out/${T}_margin_sweep.err
for s in $2; do
  env NC_TUNING=1 $(echo $s | tr ',' ' ') timeout 300 python tools/margin_sweep.py "$s" >> $O 2>> gpurun_out/${T}_margin_sweep.err
done
echo done
