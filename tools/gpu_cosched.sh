# n-tile CTAs of one A tile launched as a cluster (co-scheduling, no multicast).
set -x
mkdir -p gpurun_out
RFGPU_OZAKI_COSCHED=7 timeout 900 python -m pytest tests/test_gpu_ozaki.py -x -q > gpurun_out/pytest_cos.log 2>&1; echo "pytest exit $?"
tail -1 gpurun_out/pytest_cos.log
run_exp() {  # name, env...
  env "${@:2}" timeout 400 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp cos2 RFGPU_OZAKI_COSCHED=2
run_exp cos3 RFGPU_OZAKI_COSCHED=3
run_exp base
run_exp cos2b RFGPU_OZAKI_COSCHED=2
run_exp cos3b RFGPU_OZAKI_COSCHED=3
run_exp baseb
RFGPU_OZAKI_COSCHED=3 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:ozaki_gemm -c 6 --csv python bench.py --no-e2e --no-cpu-baseline --steps 1 --warmup 0 > gpurun_out/ncu_cos.csv 2>gpurun_out/ncu_cos.err; echo "ncu exit $?"
