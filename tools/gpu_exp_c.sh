#!/bin/bash
# experiment batch C: plane-granular ring A/B, co-scheduled n-tile clusters
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ozaki.py -m gpu -q -x > gpurun_out/expC_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/expC_pytest.log
for i in 1 2; do
RFGPU_OZAKI_FINE=0 timeout 300 python tools/pass_exp.py >> gpurun_out/expC_pass.txt 2>&1
timeout 300 python tools/pass_exp.py >> gpurun_out/expC_pass.txt 2>&1
done
RFGPU_OZAKI_COSCHED=4 timeout 300 python tools/pass_exp.py >> gpurun_out/expC_pass.txt 2>&1
RFGPU_OZAKI_COSCHED=2 timeout 300 python tools/pass_exp.py >> gpurun_out/expC_pass.txt 2>&1
RFGPU_OZAKI_FINE=0 RFGPU_OZAKI_COSCHED=4 timeout 300 python tools/pass_exp.py >> gpurun_out/expC_pass.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_rsvd.py tests/test_gpu_configs.py -m gpu -q -x >> gpurun_out/expC_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/expC_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/expC_bench_c3.json 2> gpurun_out/expC_bench_c3.err
