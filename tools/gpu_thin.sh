set -x
mkdir -p gpurun_out
run_exp() {  # name, env...
  env "${@:2}" timeout 500 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp thinp
run_exp thinnp RFGPU_OZAKI_THIN_PERSIST=0
run_exp dmma RFGPU_DIGIT_GRAM=0
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ozaki_gemm" --csv --log-file gpurun_out/l_thin.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu exit $?"
timeout 600 python -m pytest tests/test_gpu_rsvd.py tests/test_gpu_ozaki.py -x -q > gpurun_out/pytest_part.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_part.log
