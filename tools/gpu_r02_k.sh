#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "" "RFGPU_OZAKI_EQ48=1" "RFGPU_OZAKI_EQ48=2"; do
  env $v timeout 300 python tools/pass_exp.py >> gpurun_out/r02k_passexp.txt 2>&1
done
RFGPU_OZAKI_EQ48=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second -k regex:ozaki_gemm_kernel -c 12 python tools/pass_exp.py > gpurun_out/r02k_ncu_eq48.txt 2>&1
for v in "" "RFGPU_OZAKI_EQ48=1"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/r02k_bench.jsonl 2>/dev/null
done
