#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python bench.py --workload c3plain --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/expH2_bench_c3plain.json 2> gpurun_out/expH2_bench_c3plain.err
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/expH2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/expH2_pytest.log
timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/expH2_bench_c4.json 2> gpurun_out/expH2_bench_c4.err
