#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/r02c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02c_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02c_bench_c3.json 2> gpurun_out/r02c_bench_c3.err
for wl in c1 c2 c3plain c4stream; do timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02c_bench_$wl.json 2> gpurun_out/r02c_bench_$wl.err; done
timeout 1800 python tools/parity_config_full.py c4 > gpurun_out/r02c_parity_c4.log 2>&1
cp profiles/r02_parity_c4.json tests/golden/config_golden.json gpurun_out/ 2>/dev/null
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 50 python tools/sanitize_calls.py > gpurun_out/r02c_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/r02c_memcheck.log
