set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01_c1.csv python bench.py --workload c1 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "exit $?"
