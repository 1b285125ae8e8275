# A/B on one box: build, the given GPU tests, then bench.py (no solve) with the default and with each listed
# grid-kernel variant.  usage (under gpurun): bash tools/gpu_ab.sh <tag> "<pytest args or empty>" "<variant> <variant> ..."
cd $GRAFT_REPO_ROOT
T=$1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/${T}_build.log; exit 1; }
if [ -n "$2" ]; then
  timeout 1500 python -m pytest $2 -m gpu -x -q --durations=10 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
  tail -3 gpurun_out/${T}_pytest_gpu.log
fi
i=0
for v in default $3; do
  if [ "$v" = default ]; then E=""; else E="NC_TUNING=1 NC_GRID_VARIANT=$v"; fi
  env $E timeout 900 python bench.py --no-cpu-baseline --no-solve > gpurun_out/${T}_bench$i.json 2> gpurun_out/${T}_bench$i.err
  python -c "import json;d=json.loads(open('gpurun_out/${T}_bench$i.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$v',round(d['value'],3),round(d['stages_ms']['grid_pairs'],3),round(d['stages_ms']['hier_rest'],3),round(r['frac'],4),round(r['instruction_mix_bound']['cycles_per_warp_pair_isolated'],2),round(r['instruction_mix_bound']['kernel_cycles_per_warp_pair'],2))"
  i=$((i+1))
done
echo done
