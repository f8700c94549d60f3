python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:jacobi -c 1 -o gpurun_out/jacobi_c3 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_j.log 2>&1
tail -n 2 gpurun_out/ncu_j.log
