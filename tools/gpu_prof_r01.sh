# Round-1 measurement set: bench line, ncu launch list, ncu --set full of the GEMM launches.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_r01_c3.json 2> gpurun_out/bench_r01_c3.err
tail -c 4000 gpurun_out/bench_r01_c3.json
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01_c3.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"ozaki_gemm|slice_a_kernel|stats_kernel" -c 4 \
    -o gpurun_out/top_r01_c3 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out/
