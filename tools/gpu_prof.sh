# Profile set: decision trace, bench line, ncu launch list of one step, ncu --set full of the top kernels.
set -x
mkdir -p gpurun_out
RFGPU_DEBUG=1 timeout 300 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/dbg.json 2> gpurun_out/dbg.err; echo "dbg exit $?"
grep "rfgpu\]" gpurun_out/dbg.err | sort | uniq -c | head -20
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench exit $?"
tail -c 2500 gpurun_out/bench_c3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ozaki_gemm|slice_a_kernel|stats_kernel" -c 4 \
    -o gpurun_out/top_c3 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?"
ls -la gpurun_out/
