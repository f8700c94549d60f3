#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for sp in 1 0; do
  export RFGPU_SPECULATE=$sp RFGPU_DEBUG=1 RFGPU_DEBUG_PTR=1 CUDA_LAUNCH_BLOCKING=1
  P=$((29500 + sp))
  timeout 300 python tests/dist_worker.py 0 2 $P /tmp/o0.json exact_rank > gpurun_out/dbg_dist_r0_s$sp.log 2>&1 &
  timeout 300 python tests/dist_worker.py 1 2 $P /tmp/o1.json exact_rank > gpurun_out/dbg_dist_r1_s$sp.log 2>&1
  wait
  cat /tmp/o0.json /tmp/o1.json >> gpurun_out/dbg_dist_r0_s$sp.log 2>/dev/null
done
