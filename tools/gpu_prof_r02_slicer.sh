#!/bin/bash
# ncu --set full of the statistics + slicing kernels of one config-3 step (same command as tools/gpu_prof_r02.sh)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export RFGPU_GRAPH=0
timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/ncu_slicer_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"slice_at_async_kernel|stats_kernel" -s 6 -c 2 \
  -o gpurun_out/slicer_r02_c3 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/ncu_slicer_r02.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_slicer_r02.log
