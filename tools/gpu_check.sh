# one GPU round trip: build, GPU tests, smoke, bench, ncu launch list + one --set full capture of the top kernel
# usage (under gpurun): bash tools/gpu_check.sh <tag> [kernel-regex]
cd $GRAFT_REPO_ROOT
T=${1:-chk}; KR=${2:-k_pairs_grid}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
CMD="python bench.py --steps 1 --warmup 1 --no-solve --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/${T}_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_launch.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KR -s 1 -c 1 -o gpurun_out/${T}_prof $CMD > gpurun_out/${T}_ncu_full.log 2>&1
echo done
