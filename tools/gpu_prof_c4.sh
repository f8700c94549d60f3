# C4 (single pass, FP32 A) launch list of one timed step.
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --workload c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_c4.log 2>&1; echo "plain exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01_c4.csv \
    python bench.py --workload c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_c4.log 2>&1; echo "ncu launches exit $?"
timeout 600 python bench.py --workload c4 --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_r01_c4.json 2> gpurun_out/bench_r01_c4.err; echo "bench exit $?"
timeout 600 python bench.py --workload c5 --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_r01_c5.json 2> gpurun_out/bench_r01_c5.err; echo "bench c5 exit $?"
