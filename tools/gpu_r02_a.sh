#!/bin/bash
# round-2 first GPU pass: full GPU suite (incl. world-2 + config-size parity), one-off full-size parity, bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -s -p no:randomly > gpurun_out/r02a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02a_pytest.log
grep "config parity" gpurun_out/r02a_pytest.log > gpurun_out/r02a_config_parity.txt
timeout 1500 python tools/parity_config_full.py c3 c5 c2 > gpurun_out/r02a_parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/r02a_parity.log
cp profiles/r02_parity_*.json tests/golden/config_golden.json gpurun_out/ 2>/dev/null
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; echo "bench rc=$?" >> gpurun_out/r02a_bench.err
