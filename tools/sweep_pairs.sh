#!/bin/bash
# pair-kernel variant sweep (direct C2 and hier C3): NC_PAIR_STAGE x NC_PAIR_TPT
for st in smem ldg; do
  for tpt in 1 2; do
    echo "stage=$st tpt=$tpt"
    NC_PAIR_STAGE=$st NC_PAIR_TPT=$tpt python bench.py --config C2 --steps 3 --warmup 2 --no-solve --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  C2 direct ms', d['ms_per_step'], d['roofline']['frac'])"
  done
  NC_PAIR_STAGE=$st python tools/hier_probe.py C3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  C3 hier ms', d['stats']['ms_last'][4], d['stats']['ms_last'][5])"
done
