# ncu --set full of the step-4 interpolation kernel (k_interp) at C5 (GPU box); source-level view for the hot loop
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pi2_build.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --no-solve --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/pi2_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_interp$" -s 1 -c 1 -o gpurun_out/pi2_prof $CMD > gpurun_out/pi2_ncu.log 2>&1
echo done
