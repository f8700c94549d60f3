python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/bench_pass_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_f64_tma -c 5 -o gpurun_out/pass_c3_v2 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_pass.log 2>&1
tail -n 2 gpurun_out/ncu_pass.log
