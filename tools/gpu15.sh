python bench.py --workload c5 --no-e2e --no-cpu-baseline --steps 1 --warmup 1 > gpurun_out/c5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cpqr_kernel -c 1 -o gpurun_out/cpqr_c5 python bench.py --workload c5 --no-e2e --no-cpu-baseline --steps 1 --warmup 1 > gpurun_out/ncu_cpqr.log 2>&1
tail -n 2 gpurun_out/ncu_cpqr.log
