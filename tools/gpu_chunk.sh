set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 > gpurun_out/exp_full.json 2> gpurun_out/exp_full.err; echo "full exit $?"
python -c "
import json; d=json.loads(open('gpurun_out/exp_full.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'], d['clocks'], {k: round(v,2) for k,v in d['phase_ms_per_step'].items() if v})"
for w in c4 c5; do
  timeout 500 python bench.py --workload $w --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$w.json 2>gpurun_out/exp_$w.err; echo "$w exit $?"
  python -c "import json; d=json.loads(open('gpurun_out/exp_$w.json').read().strip().splitlines()[-1]); print('$w', d['value'], {k: round(v,2) for k,v in d['phase_ms_per_step'].items() if v})"
done
