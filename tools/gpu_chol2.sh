set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"chol_kernel" --csv --log-file gpurun_out/l_chol.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu exit $?"
for w in c3 c2 c1; do
  timeout 500 python bench.py --workload $w --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$w.json 2>gpurun_out/exp_$w.err; echo "$w exit $?"
  python -c "import json; d=json.loads(open('gpurun_out/exp_$w.json').read().strip().splitlines()[-1]); print('$w', round(d['value']*1e3,2), {k: round(v,2) for k,v in d['phase_ms_per_step'].items() if k in ('chol','orth','small_svd')})"
done
