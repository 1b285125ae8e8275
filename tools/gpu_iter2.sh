# GPU iteration with a custom ncu selection: bash tools/gpu_iter2.sh <tag> "<pytest args>" "<ncu -k/-s/-c args>"
cd $GRAFT_REPO_ROOT
T=${1:-it}; PT=${2:-tests}; NK=$3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/${T}_build.log; exit 1; }
if [ -n "$PT" ]; then
  timeout 1500 python -m pytest $PT -m gpu -x -q --durations=10 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
  tail -3 gpurun_out/${T}_pytest_gpu.log
fi
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python -c "import json;d=json.loads(open('gpurun_out/${T}_bench.json').read().strip().splitlines()[-1]);print('bench',d['value'],d['e2e']['value'],d['stages_ms'])"
if [ -n "$NK" ]; then
  CMD="python bench.py --steps 1 --warmup 1 --no-solve --no-cpu-baseline"
  timeout 900 ncu --set full --clock-control none --import-source on $NK -o gpurun_out/${T}_prof $CMD > gpurun_out/${T}_ncu_full.log 2>&1
  echo "ncu rc=$?"
fi
echo done
