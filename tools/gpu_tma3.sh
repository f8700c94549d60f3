set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ozaki.py -x -q > gpurun_out/pytest_oz.log 2>&1; echo "pytest oz exit $?"; tail -2 gpurun_out/pytest_oz.log
run_exp() {  # name, env...
  env "${@:2}" timeout 500 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp tma3
run_exp tma2 RFGPU_OZAKI_TMA3=0
run_exp tma3b
run_exp tma3_bk32 RFGPU_OZAKI_BK=32
run_exp tma2b RFGPU_OZAKI_TMA3=0
