cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5_build.log 2>&1
timeout 2000 python tools/sweep_grid.py C5 "128,2,4,256,1,0,8" "128,2,4,256,1,0,4" "128,2,4,256,1,0,6" "256,1,4,256,1,0,1" "256,1,4,256,1,0,5" "256,1,4,256,1,0,6" "256,1,2,256,1,0,6" "256,2,2,256,1,0,5" "256,1,4,128,1,1,6" "128,2,4,128,1,1,8" "256,1,4,512,1,0,5" > gpurun_out/s5_sweep_c5.jsonl 2>&1
echo done
