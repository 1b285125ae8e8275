cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pi_build.log 2>&1
timeout 900 python -m pytest tests/test_multirank_emulated_gpu.py tests/test_hier_gpu.py -x -q -k "emulated or C2" > gpurun_out/pi_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pi_pytest.log
CMD="python bench.py --steps 1 --warmup 1 --no-solve --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/pi_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_interp" -s 1 -c 1 -o gpurun_out/pi_prof $CMD > gpurun_out/pi_ncu.log 2>&1
echo done
