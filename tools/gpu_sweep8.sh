cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s8_build.log 2>&1
for c in C3 C4 C5; do NC_HIER_DIAG=1 timeout 300 python tools/hier_probe.py $c > gpurun_out/s8_diag_$c.log 2>&1; done
timeout 900 python tools/sweep_grid.py C5 "128,2,4,256,0,0,8" "128,2,4,256,1,0,8" > gpurun_out/s8_sweep_c5.jsonl 2>&1
CMD="python bench.py --config C4 --steps 1 --warmup 1 --no-solve --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/s8_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_interp|k_pairs_near|k_transform" -s 3 -c 3 -o gpurun_out/s8_prof_rest $CMD > gpurun_out/s8_ncu.log 2>&1
echo done
