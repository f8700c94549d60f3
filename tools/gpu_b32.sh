set -x
mkdir -p gpurun_out
for w in c1 c2; do
  for b in 4 8; do
  RFGPU_JACOBI_BLOCK=$b RFGPU_DEBUG=1 timeout 500 python bench.py --workload $w --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/exp_$w.json 2>gpurun_out/exp_$w.err; echo "$w exit $?"
  python -c "import json; d=json.loads(open('gpurun_out/exp_$w.json').read().strip().splitlines()[-1]); print('$w B=$b', round(d['value']*1e3,3), {k: round(v,3) for k,v in d['phase_ms_per_step'].items() if k in ('jacobi','small_svd')})"
  grep "sweeps" gpurun_out/exp_$w.err | sort | uniq -c | head -2
  done
done
RFGPU_JACOBI_BLOCK=4 timeout 900 python -m pytest tests/test_gpu_rsvd.py -x -q > gpurun_out/pytest_b32.log 2>&1; echo "pytest b32 exit $?"; tail -1 gpurun_out/pytest_b32.log
