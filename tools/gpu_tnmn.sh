set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ozaki.py -x -q > gpurun_out/pytest_oz.log 2>&1; echo "pytest oz exit $?"; tail -3 gpurun_out/pytest_oz.log
run_exp() {  # name, env...
  env "${@:2}" timeout 400 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp tnmn
run_exp tnkm RFGPU_OZAKI_TNMN=0
run_exp tnmn_mc0 RFGPU_OZAKI_MC=0
run_exp tnmn_tnk4k_mc0 RFGPU_OZAKI_MC=0 RFGPU_OZAKI_TNK=4096
run_exp tnmn2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
