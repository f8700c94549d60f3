set -x
python bench.py > gpurun_out/bench_r01_c3.json 2> gpurun_out/bench_r01_c3.err
tail -c 3000 gpurun_out/bench_r01_c3.json
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rfgpu --csv --log-file gpurun_out/launches_r01_c3.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_f64_tma -c 6 -o gpurun_out/top_r01_c3 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out/
