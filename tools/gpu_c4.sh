set -x
mkdir -p gpurun_out
for w in c4 c3 c5; do
  RFGPU_DEBUG=1 timeout 600 python bench.py --workload $w --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/exp_$w.json 2> gpurun_out/exp_$w.err; echo "$w exit $?"
  python -c "import json; d=json.loads(open('gpurun_out/exp_$w.json').read().strip().splitlines()[-1]); print('$w', d['value'], {k: round(v,2) for k,v in d['phase_ms_per_step'].items() if v})"
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
