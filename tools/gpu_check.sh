# Round-1 GPU session: parity tests, smoke, stage-depth / multicast / persistence experiments, bench.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_gpu.log
RFGPU_OZAKI_BK=32 timeout 600 python -m pytest tests/test_gpu_ozaki.py -x -q > gpurun_out/pytest_bk32.log 2>&1; echo "pytest bk32 exit $?"
tail -3 gpurun_out/pytest_bk32.log
RFGPU_OZAKI_PERSIST=0 RFGPU_OZAKI_FUSED=0 timeout 600 python -m pytest tests/test_gpu_ozaki.py -x -q > gpurun_out/pytest_np.log 2>&1; echo "pytest nopersist nofused exit $?"
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -3 gpurun_out/smoke.log
run_exp() {  # name, env...
  env "${@:2}" timeout 400 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python -c "
import json; d=json.loads(open('gpurun_out/exp_$1.json').read().strip().splitlines()[-1]); ph=d['phase_ms_per_step']; print('$1', round(d['value']*1e3,2), 'nn', round(ph['pass_nn'],2), 'tn', round(ph['pass_tn'],2), 'slice', round(ph['ozaki_slice'],2), 'orth', round(ph['orth'],2), 'svd', round(ph['small_svd'],2), 'clk', d.get('clocks'))"
}
run_exp base
run_exp nopersist RFGPU_OZAKI_PERSIST=0
run_exp bk32 RFGPU_OZAKI_BK=32
run_exp bk32_mc1 RFGPU_OZAKI_BK=32 RFGPU_OZAKI_MC=1
run_exp bk32_mc0 RFGPU_OZAKI_BK=32 RFGPU_OZAKI_MC=0
run_exp mc1 RFGPU_OZAKI_MC=1
run_exp mc0 RFGPU_OZAKI_MC=0
run_exp twosets RFGPU_OZAKI_SHARED=0
run_exp nofused RFGPU_OZAKI_FUSED=0
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench exit $?"
tail -c 3000 gpurun_out/bench_c3.json
