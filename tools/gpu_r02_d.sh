#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/r02d_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02d_pytest.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/r02d_bench_c3.json 2> gpurun_out/r02d_bench_c3.err
for wl in c1 c3plain c4stream; do timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02d_bench_$wl.json 2> gpurun_out/r02d_bench_$wl.err; done
for v in "" "RFGPU_OZAKI_ILV=1" "RFGPU_OZAKI_ILV=1 RFGPU_OZAKI_MC=1 RFGPU_OZAKI_MCSIZE=2"; do
  env $v timeout 300 python tools/pass_exp.py >> gpurun_out/r02d_passexp.txt 2>&1
done
bash tools/gpu_prof_r02.sh
