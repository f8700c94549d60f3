# Epilogue warps wait for the accumulator with a suspend-time hint.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py -x -q > gpurun_out/pytest_sleep.log 2>&1; echo "pytest exit $?"
tail -2 gpurun_out/pytest_sleep.log
timeout 600 python tools/tile_overhead.py > gpurun_out/tile_sleep.txt 2>&1; echo "tile exit $?"
tail -2 gpurun_out/tile_sleep.txt
run_exp() {  # name, env...
  env "${@:2}" timeout 400 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp sleep1
run_exp sleep2
