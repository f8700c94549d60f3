#!/bin/bash
# ncu evidence for round 2 (config 3): launch list of identical eager steps and a --set full capture of one
# step's digit-GEMM launches. Each command only after the same command ran clean without ncu (bench runs).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export RFGPU_GRAPH=0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_r02_c3.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/ncu_launch_r02.log 2>&1
echo "launch rc=$?" >> gpurun_out/ncu_launch_r02.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:ozaki_gemm_kernel -s 21 -c 7 \
  -o gpurun_out/top_r02_c3 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/ncu_full_r02.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full_r02.log
