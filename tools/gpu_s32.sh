# fp32 SFU seeds in the far form (R31): loop-body microbench, C5/C4 grid-kernel time and C3/C4 hier-vs-direct error
# (historical: FAR 7/8 were instantiated for this measurement only and removed after it; profiles/r01w_s32.txt)
# per FAR variant (5 = fp64 MUFU seeds, 7 = both seeds fp32, 8 = rsqrt seed fp32)  (GPU box)
cd $GRAFT_REPO_ROOT
T=${1:-s32}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1906_04209_b200/csrc -o /tmp/pmb tools/pair_mix_bench.cu && /tmp/pmb > gpurun_out/${T}_pair_mix.txt 2>&1
timeout 900 python tools/sweep_grid.py C5 "8,2,4,64,5,3,3" "8,2,4,64,7,3,3" "8,2,4,64,8,3,3" "8,2,4,64,5,3,3" "8,2,4,64,7,3,3" > gpurun_out/${T}_sweep_c5.jsonl 2>&1
timeout 600 python tools/sweep_grid.py C4 "8,2,4,64,5,3,3" "8,2,4,64,7,3,3" "8,2,4,64,8,3,3" > gpurun_out/${T}_sweep_c4.jsonl 2>&1
for v in "8,2,4,64,5,3,3" "8,2,4,64,7,3,3" "8,2,4,64,8,3,3"; do
  for c in C3 C4; do
    NC_GRID_VARIANT=$v timeout 600 python tools/hier_accuracy.py $c 1e-9 | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/${T}_acc.jsonl 2>&1
  done
done
echo done
