#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/r02m_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02m_pytest.log
for wl in c3plain c2 c1; do timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02m_bench_$wl.json 2> gpurun_out/r02m_bench_$wl.err; done
timeout 2400 python tools/ref_full_time.py 8 gpurun_out/r02m_ref_c3_8threads.json > gpurun_out/r02m_ref8.log 2>&1
