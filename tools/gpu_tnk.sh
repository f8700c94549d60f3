set -x
mkdir -p gpurun_out
run_exp() {  # name, env...
  env "${@:2}" timeout 400 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp base
run_exp tnk4k_mc0 RFGPU_OZAKI_TNK=4096 RFGPU_OZAKI_MC=0
run_exp tnk4k_mc1 RFGPU_OZAKI_TNK=4096
run_exp tnk8k_mc0 RFGPU_OZAKI_TNK=8192 RFGPU_OZAKI_MC=0
run_exp tnk2k_mc0 RFGPU_OZAKI_TNK=2048 RFGPU_OZAKI_MC=0
run_exp tnk4k_mc0_p RFGPU_OZAKI_TNK=4096 RFGPU_OZAKI_MC=0 RFGPU_OZAKI_PERSIST=1
RFGPU_OZAKI_TNK=4096 RFGPU_OZAKI_MC=0 timeout 600 python -m pytest tests/test_gpu_ozaki.py -x -q > gpurun_out/pytest_tnk.log 2>&1; echo "pytest tnk exit $?"; tail -2 gpurun_out/pytest_tnk.log
