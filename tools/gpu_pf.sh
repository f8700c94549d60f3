set -x
mkdir -p gpurun_out
run_exp() {  # name, env...
  env "${@:2}" timeout 500 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp pf0
run_exp pf2 RFGPU_OZAKI_PF=2
run_exp pf4 RFGPU_OZAKI_PF=4
run_exp pf8 RFGPU_OZAKI_PF=8
run_exp pf0b
RFGPU_OZAKI_PF=4 timeout 600 python -m pytest tests/test_gpu_ozaki.py -x -q > gpurun_out/pytest_pf.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/pytest_pf.log
