# ncu --set full with source of one chol_kernel launch (config 3, l = 220).
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chol_kernel -c 1 -o gpurun_out/chol_full python bench.py --no-e2e --no-cpu-baseline --steps 1 --warmup 0 > gpurun_out/ncu_cholfull.log 2>&1; echo "ncu exit $?"
ls -la gpurun_out/chol_full.ncu-rep
