set -x
mkdir -p gpurun_out
RFGPU_OZAKI_KINNER=1 timeout 600 python -m pytest tests/test_gpu_ozaki.py -x -q > gpurun_out/pytest_kin.log 2>&1; echo "pytest kin exit $?"; tail -1 gpurun_out/pytest_kin.log
run_exp() {  # name, env...
  env "${@:2}" timeout 500 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp kout
run_exp kin RFGPU_OZAKI_KINNER=1
run_exp kout2
run_exp kin2 RFGPU_OZAKI_KINNER=1
