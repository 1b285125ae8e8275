# one GPU iteration: build, selected GPU tests (with durations), bench (no cpu baseline), optional ncu --set full of one kernel
# usage (under gpurun): bash tools/gpu_iter.sh <tag> "<pytest args>" [kernel-regex]
cd $GRAFT_REPO_ROOT
T=${1:-it}; PT=${2:-tests}; KR=$3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1500 python -m pytest $PT -m gpu -x -q --durations=20 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
tail -3 gpurun_out/${T}_pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python -c "import json;d=json.loads(open('gpurun_out/${T}_bench.json').read().strip().splitlines()[-1]);print('bench',d['value'],d['e2e']['value'],d['stages_ms'])"
if [ -n "$KR" ]; then
  CMD="python bench.py --steps 1 --warmup 1 --no-solve --no-cpu-baseline"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KR -s ${NCU_SKIP:-1} -c 1 -o gpurun_out/${T}_prof $CMD > gpurun_out/${T}_ncu_full.log 2>&1
  echo "ncu rc=$?"
fi
echo done
