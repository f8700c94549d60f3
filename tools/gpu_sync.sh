set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_rsvd.py -x -q > gpurun_out/pytest_part.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_part.log
run_exp() {  # name, env...
  env "${@:2}" timeout 500 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp nosync
run_exp nosync2
timeout 600 python bench.py --steps 3 > gpurun_out/exp_full.json 2> gpurun_out/exp_full.err; echo "full exit $?"; tail -c 600 gpurun_out/exp_full.json
