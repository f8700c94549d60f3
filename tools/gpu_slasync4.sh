# FP32 cp.async slicer: full GPU tests, then A/B at config 4.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_sla4.log 2>&1; echo "pytest exit $?"
tail -2 gpurun_out/pytest_sla4.log
run_exp() {  # name, env...
  env "${@:2}" timeout 400 python bench.py --workload c4 --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp c4async
run_exp c4regs RFGPU_OZAKI_SLICE_ASYNC=0
run_exp c4async2
run_exp c4regs2 RFGPU_OZAKI_SLICE_ASYNC=0
