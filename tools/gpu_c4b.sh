set -x
mkdir -p gpurun_out
for v in a b; do
  timeout 600 python bench.py --workload c4 --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/exp_c4$v.json 2> gpurun_out/exp_c4$v.err; echo "c4 exit $?"
  python -c "import json; d=json.loads(open('gpurun_out/exp_c4$v.json').read().strip().splitlines()[-1]); print('c4$v', d['value'], d['ms_per_step'], {k: round(v,2) for k,v in d['phase_ms_per_step'].items() if v})"
done
RFGPU_JACOBI_BLOCK=0 timeout 600 python bench.py --workload c4 --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/exp_c4c.json 2> gpurun_out/exp_c4c.err; echo "c4 exit $?"
python -c "import json; d=json.loads(open('gpurun_out/exp_c4c.json').read().strip().splitlines()[-1]); print('c4c', d['value'], {k: round(v,2) for k,v in d['phase_ms_per_step'].items() if v})"
