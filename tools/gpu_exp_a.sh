#!/bin/bash
# experiment batch A: INT8 peaks, MMA chunking A/B, fold parity, c3 phases
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python tools/i8_peaks.py gpurun_out/expA_i8_peaks.json > gpurun_out/expA_i8_peaks.log 2>&1
for i in 1 2; do
RFGPU_OZAKI_CHUNK=0 timeout 300 python tools/pass_exp.py >> gpurun_out/expA_pass.txt 2>&1
timeout 300 python tools/pass_exp.py >> gpurun_out/expA_pass.txt 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_rsvd.py tests/test_gpu_ozaki.py tests/test_gpu_configs.py tests/test_gpu_dist_world2.py tests/test_gpu_graph.py -m gpu -q -x > gpurun_out/expA_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/expA_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/expA_bench_c3.json 2> gpurun_out/expA_bench_c3.err
timeout 300 python bench.py --workload c2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/expA_bench_c2.json 2> gpurun_out/expA_bench_c2.err
