# quick GPU round trip: build, all GPU tests, bench (no ncu).  usage: bash tools/gpu_quick.sh <tag> [bench args]
cd $GRAFT_REPO_ROOT
T=${1:-q}; shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline "$@" > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo done
