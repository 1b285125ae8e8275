# grid-tolerance factor sweep (R21): hier-vs-direct error at C3/C4, difference from factor 100 at C5, times
# usage (under gpurun): bash tools/gpu_tol_sweep.sh <tag>
cd $GRAFT_REPO_ROOT
T=${1:-tol}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
NC_TUNING=1 timeout 1500 python tools/env_sweep.py --settings '[["f100", {"NC_GRID_TOL_FACTOR": "100"}], ["f1000", {}], ["f1500", {"NC_GRID_TOL_FACTOR": "1500"}], ["f2000", {"NC_GRID_TOL_FACTOR": "2000"}], ["f2500", {"NC_GRID_TOL_FACTOR": "2500"}], ["f3000", {"NC_GRID_TOL_FACTOR": "3000"}]]' C3 C4 C5 > gpurun_out/${T}_tol_sweep.jsonl 2> gpurun_out/${T}_tol_sweep.err
echo done
