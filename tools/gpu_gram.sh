set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
run_exp() {  # name, env...
  env "${@:2}" timeout 500 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp dgram
run_exp dmmagram RFGPU_DIGIT_GRAM=0
run_exp dgram2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"slice_at|ozaki_gemm|reduce_ws|slice_r|col_exp" --csv --log-file gpurun_out/l_gram.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu exit $?"
