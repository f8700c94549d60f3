set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_rsvd.py -x -q > gpurun_out/pytest_part.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/pytest_part.log
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"slice_at" --csv --log-file gpurun_out/l_s2.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu exit $?"
run_exp() {  # name, env...
  env "${@:2}" timeout 500 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp s2
run_exp s2b
