#!/bin/bash
# experiment batch B: MMA chunking A/B (compile-time tables), TMA-only / MMA-only / no-B-load pass variants
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for i in 1 2; do
RFGPU_OZAKI_CHUNK=0 timeout 300 python tools/pass_exp.py >> gpurun_out/expB_pass.txt 2>&1
timeout 300 python tools/pass_exp.py >> gpurun_out/expB_pass.txt 2>&1
done
for mode in 1 2 3; do
RFGPU_OZAKI_EXP=$mode timeout 300 python tools/pass_exp.py >> gpurun_out/expB_pass.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_rsvd.py -m gpu -q -x > gpurun_out/expB_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/expB_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/expB_bench_c3.json 2> gpurun_out/expB_bench_c3.err
RFGPU_OZAKI_CHUNK=0 timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/expB_bench_c3_chunk0.json 2> gpurun_out/expB_bench_c3_chunk0.err
