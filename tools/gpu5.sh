python tools/prof_small.py > gpurun_out/prof_small_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:jacobi -s 1 -c 1 -o gpurun_out/jacobi110 python tools/prof_small.py > gpurun_out/ncu_jacobi.log 2>&1
python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/bench_pass_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_f64_kernel -c 2 -o gpurun_out/pass_c3 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_pass.log 2>&1
tail -3 gpurun_out/ncu_jacobi.log gpurun_out/ncu_pass.log
