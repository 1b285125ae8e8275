cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s12_build.log 2>&1
timeout 900 python tools/sweep_grid.py C5 "NC_INTERP_VARIANT=128,4,1" "NC_INTERP_VARIANT=0,0,0" > gpurun_out/s12_sweep_c5.jsonl 2>&1
CMD="python bench.py --config C4 --steps 1 --warmup 1 --no-solve --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/s12_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_interp" -s 1 -c 1 -o gpurun_out/s12_prof_interp $CMD > gpurun_out/s12_ncu.log 2>&1
echo done
