set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
for w in c3 c2 c1 c4; do
  RFGPU_DEBUG=1 timeout 500 python bench.py --workload $w --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$w.json 2>gpurun_out/exp_$w.err; echo "$w exit $?"
  python -c "import json; d=json.loads(open('gpurun_out/exp_$w.json').read().strip().splitlines()[-1]); print('$w', round(d['value']*1e3,2), {k: round(v,2) for k,v in d['phase_ms_per_step'].items() if k in ('jacobi','small_svd','single_pass_core')})"
  grep "sweeps" gpurun_out/exp_$w.err | sort | uniq -c | head -3
done
