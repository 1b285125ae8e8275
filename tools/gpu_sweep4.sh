cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4_build.log 2>&1
timeout 1500 python tools/sweep_grid.py C5 "2,4,0,256,1,0,1" "2,1,0,256,1,0,4" "2,1,0,256,1,0,2" "2,2,0,256,1,0,2" "1,1,0,256,1,0,4" "1,1,0,256,1,0,8" "1,2,0,256,1,0,4" "1,1,0,128,1,0,4" > gpurun_out/s4_sweep_c5.jsonl 2>&1
echo done
