#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
RFGPU_DEBUG=1 timeout 300 python tools/jac_bench.py > gpurun_out/expG_jac.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/expG_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/expG_pytest.log
for wl in c1 c2 c4 c3 c5; do
  timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/expG_bench_${wl}.json 2> gpurun_out/expG_bench_${wl}.err
done
