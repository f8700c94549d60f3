# Round-1 GPU session: parity tests, smoke, stage-depth / multicast experiments, bench.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_gpu.log
RFGPU_OZAKI_BK=32 timeout 600 python -m pytest tests/test_gpu_ozaki.py -x -q > gpurun_out/pytest_bk32.log 2>&1; echo "pytest bk32 exit $?"
tail -3 gpurun_out/pytest_bk32.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -3 gpurun_out/smoke.log
for bk in 64 32; do for mc in unset 0 1; do
  if [ $mc = unset ]; then unset RFGPU_OZAKI_MC; else export RFGPU_OZAKI_MC=$mc; fi
  RFGPU_OZAKI_BK=$bk timeout 400 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_bk${bk}_mc${mc}.json 2>gpurun_out/exp_bk${bk}_mc${mc}.err
  echo "bk=$bk mc=$mc exit $?"; python -c "
import json,sys; d=json.loads(open('gpurun_out/exp_bk${bk}_mc${mc}.json').read().strip().splitlines()[-1]); print(d['value'], d['phase_ms_per_step'])" 
done; done
unset RFGPU_OZAKI_MC
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench exit $?"
tail -c 3000 gpurun_out/bench_c3.json
