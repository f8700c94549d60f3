# Round-1 measurement set: bench line, ncu launch list of one step, ncu --set full of the top kernels (config 3).
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_r01_c3.json 2> gpurun_out/bench_r01_c3.err; echo "bench exit $?"
tail -c 2500 gpurun_out/bench_r01_c3.json
timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1; echo "plain exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01_c3.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"ozaki_gemm|slice_at|stats_kernel" -c 6 \
    -o gpurun_out/top_r01_c3 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/smoke.log
ls -la gpurun_out/
