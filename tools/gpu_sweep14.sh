cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s14_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s14_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s14_pytest.log
timeout 900 python tools/sweep_grid.py C5 "NC_INTERP_VARIANT=128,4,1" "NC_INTERP_VARIANT=256,2,1" "NC_INTERP_VARIANT=512,1,1" "NC_INTERP_VARIANT=256,1,4" "NC_INTERP_VARIANT=256,2,4" > gpurun_out/s14_sweep_c5.jsonl 2>&1
timeout 600 python bench.py --config C2 --mode direct --no-cpu-baseline --no-solve > gpurun_out/s14_bench_c2.json 2> gpurun_out/s14_bench_c2.err
echo done
