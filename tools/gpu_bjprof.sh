set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bjacobi" -c 1 -o gpurun_out/bj_full python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/bj_f.log 2>&1; echo "exit $?"
