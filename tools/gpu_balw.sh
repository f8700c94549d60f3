# Balanced n-tile widths (l = 220: 64 64 48 48) against 64 64 64 32.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_rsvd.py -x -q > gpurun_out/pytest_balw.log 2>&1; echo "pytest exit $?"
tail -2 gpurun_out/pytest_balw.log
RFGPU_OZAKI_NARROW=1 timeout 900 python -m pytest tests/test_gpu_ozaki.py -x -q > gpurun_out/pytest_balw1.log 2>&1; echo "pytest narrow1 exit $?"
tail -1 gpurun_out/pytest_balw1.log
run_exp() {  # name, env...
  env "${@:2}" timeout 400 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp balw
run_exp last RFGPU_OZAKI_NARROW=1
run_exp balw2
run_exp last2 RFGPU_OZAKI_NARROW=1
