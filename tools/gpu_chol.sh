set -x
mkdir -p gpurun_out
run_exp() {  # name, env...
  env "${@:2}" timeout 400 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp chol_new
run_exp chol_old RFGPU_CHOL=0
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
run_exp chol_new2
