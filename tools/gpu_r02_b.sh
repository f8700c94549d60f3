#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/r02b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_pytest.log
for v in "" "RFGPU_OZAKI_MC=1 RFGPU_OZAKI_MCSIZE=2" "RFGPU_OZAKI_MC=1 RFGPU_OZAKI_MCSIZE=4"; do
  env $v timeout 300 python tools/pass_exp.py >> gpurun_out/r02b_passexp.txt 2>&1
done
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02b_bench_c3.json 2> gpurun_out/r02b_bench_c3.err
for wl in c1 c2 c4 c5; do timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02b_bench_$wl.json 2> gpurun_out/r02b_bench_$wl.err; done
timeout 900 python tools/probe_ref_timing.py 32768,65536,131072,262144 16 gpurun_out/r02b_refcurve16.json > /dev/null 2>&1
timeout 600 python tools/probe_ref_timing.py 65536,131072 8 gpurun_out/r02b_refcurve8.json > /dev/null 2>&1
