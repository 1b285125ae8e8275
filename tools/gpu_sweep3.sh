cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s3_build.log 2>&1
timeout 1500 python tools/sweep_grid.py C5 "2,4,0,256,1,0" "2,4,0,128,1,1" "2,4,0,256,1,1" "2,2,0,128,1,1" "2,4,0,64,1,1" "2,4,0,128,0,1" > gpurun_out/s3_sweep_c5.jsonl 2>&1
timeout 600 python tools/sweep_grid.py C4 "2,4,0,256,1,0" "2,4,0,128,1,1" > gpurun_out/s3_sweep_c4.jsonl 2>&1
echo done
