#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvcc -O3 -Xcompiler -mavx2 -o /tmp/hostcopy_nt tools/microbench/hostcopy_nt.cu 2>/dev/null && /tmp/hostcopy_nt > gpurun_out/expI_hostcopy_nt.txt 2>&1
grep -m1 "model name" /proc/cpuinfo >> gpurun_out/expI_hostcopy_nt.txt; nproc >> gpurun_out/expI_hostcopy_nt.txt
RFGPU_STAGE_NT=0 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/expI_bench_c3_nt0.json 2> gpurun_out/expI_bench_c3_nt0.err
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/expI_bench_c3_nt1.json 2> gpurun_out/expI_bench_c3_nt1.err
RFGPU_STAGE_NT=0 timeout 900 python bench.py --workload c4stream --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/expI_bench_c4s_nt0.json 2> gpurun_out/expI_bench_c4s_nt0.err
timeout 900 python bench.py --workload c4stream --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/expI_bench_c4s_nt1.json 2> gpurun_out/expI_bench_c4s_nt1.err
