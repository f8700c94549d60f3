#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./tools/microbench/hostcopy > gpurun_out/r02e_hostcopy.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:randomly -x > gpurun_out/r02e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02e_pytest.log
for wl in c1 c2 c3plain c4 c5; do timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02e_bench_$wl.json 2> gpurun_out/r02e_bench_$wl.err; done
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02e_bench_c3.json 2> gpurun_out/r02e_bench_c3.err
