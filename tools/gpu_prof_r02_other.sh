#!/bin/bash
# ncu --set full of the non-pass kernels of one config-3 step (slicer, statistics, DMMA GEMMs, block Jacobi, Cholesky):
# same command as tools/gpu_prof_r02.sh (which ran clean without ncu in the same call sequence)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export RFGPU_GRAPH=0
timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/ncu_other_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"slice_at_async_kernel|stats_kernel|gemm_f64_tma_kernel|bjacobi_kernel|chol_kernel|slice_r_kernel" -s 84 -c 30 \
  -o gpurun_out/other_r02_c3 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/ncu_other_r02.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_other_r02.log
# statistics + slicing kernels of the 4th step (2 matching launches per step)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"slice_at_async_kernel|stats_kernel" -s 6 -c 2 \
  -o gpurun_out/slicer_r02_c3 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/ncu_slicer_r02.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_slicer_r02.log
# summaries: ncu -i gpurun_out/{other,slicer}_r02_c3.ncu-rep --page raw --csv -> profiles/r02_ncu_other_kernels_c3.jsonl
