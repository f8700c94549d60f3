set -x
mkdir -p gpurun_out
RFGPU_JACOBI_SORT=1 timeout 900 python -m pytest tests/test_gpu_rsvd.py tests/test_gpu_id_cur.py -x -q > gpurun_out/pytest_part.log 2>&1; echo "pytest sort exit $?"; tail -1 gpurun_out/pytest_part.log
for w in c3 c2 c1 c4; do
  for so in 0 1; do
  RFGPU_JACOBI_SORT=$so RFGPU_DEBUG=1 timeout 500 python bench.py --workload $w --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$w.json 2>gpurun_out/exp_$w.err; echo "$w exit $?"
  python -c "import json; d=json.loads(open('gpurun_out/exp_$w.json').read().strip().splitlines()[-1]); print('$w sort=$so', round(d['value']*1e3,2), {k: round(v,2) for k,v in d['phase_ms_per_step'].items() if k in ('jacobi','small_svd','single_pass_core')})"
  grep "sweeps" gpurun_out/exp_$w.err | sort | uniq -c | head -3
  done
done
