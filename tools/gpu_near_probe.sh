# near-list / rank-cut row errors, one process per setting; usage (under gpurun): bash tools/gpu_near_probe.sh <tag> "<K=V,K=V> ..." [configs]
cd $GRAFT_REPO_ROOT
T=$1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
O=gpurun_out/${T}_near_rows_probe.jsonl; : > $O
for s in $2; do
  env NC_TUNING=1 $(echo $s | tr ',' ' ') timeout 400 python tools/near_rows_probe.py "$s" $3 >> $O 2>> gpurun_out/${T}_near_rows_probe.err
done
cat $O
echo done
