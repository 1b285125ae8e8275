# step-4 interpolation: coefficient prefetch variant (k_interp MB = 3) vs the current default at C5 and C4 (GPU box)
cd $GRAFT_REPO_ROOT
T=${1:-pf}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python tools/sweep_grid.py C5 "NC_INTERP_VARIANT=128,2,0,4" "NC_INTERP_VARIANT=128,2,3,4" "NC_INTERP_VARIANT=128,2,4,4" "NC_INTERP_VARIANT=128,2,3,4" "NC_INTERP_VARIANT=128,2,4,4" > gpurun_out/${T}_sweep_c5.jsonl 2>&1
timeout 600 python tools/sweep_grid.py C4 "NC_INTERP_VARIANT=128,2,0,4" "NC_INTERP_VARIANT=128,2,3,4" "NC_INTERP_VARIANT=128,2,4,4" > gpurun_out/${T}_sweep_c4.jsonl 2>&1
echo done
