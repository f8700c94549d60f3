#!/bin/bash
# How the round-2 evidence was produced on a B200 box (gpurun: the repo copy is $GRAFT_REPO_ROOT).
#   bash tools/gpu_round2.sh [tests] [parity] [bench] [prof] [host]
# tests  : the GPU parity suite (incl. config-size parity, world-2 row sharding, graphs, edge cases, CLI)
# parity : full-size comparisons against the compiled reference on the bench's A
#          -> profiles/r02_parity_c{2,3,4,5}.json, tests/golden/config_golden.json; the reference's full config 3
#          at its default 8 threads -> profiles/r02_reference_c3_8threads.json
# bench  : every workload (config 3 with e2e and the anchored CPU baseline)
# prof   : ncu launch list + --set full of the digit GEMMs at config 3 (tools/gpu_prof_r02.sh,
#          then tools/summarize_prof.py r02 c3 5 here)
# host   : host copy bandwidths (tools/microbench/hostcopy.cu) and the reference's per-row cost curve
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for what in "${@:-tests bench}"; do
  case "$what" in
    tests)
      timeout 1800 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/round2_pytest.log 2>&1
      echo "pytest rc=$?" >> gpurun_out/round2_pytest.log ;;
    parity)
      timeout 3600 python tests/fullsize/parity_config_full.py c3 c5 c2 c4 > gpurun_out/round2_parity.log 2>&1
      cp profiles/r02_parity_*.json tests/golden/config_golden.json gpurun_out/ 2>/dev/null
      timeout 2400 python tests/fullsize/ref_full_time.py 8 gpurun_out/r02_reference_c3_8threads.json ;;
    bench)
      timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/round2_bench_c3.json 2> gpurun_out/round2_bench_c3.err
      for wl in c1 c2 c3plain c4 c4stream c5; do
        timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --no-e2e --no-cpu-baseline \
          > gpurun_out/round2_bench_$wl.json 2> gpurun_out/round2_bench_$wl.err
      done ;;
    prof)
      bash tools/gpu_prof_r02.sh ;;
    host)
      /usr/local/cuda/bin/nvcc -O3 -o /tmp/hostcopy tools/microbench/hostcopy.cu && /tmp/hostcopy > gpurun_out/round2_hostcopy.txt 2>&1
      timeout 900 python tests/fullsize/probe_ref_timing.py 32768,65536,131072,262144 16 gpurun_out/round2_refcurve16.json ;;
  esac
done
