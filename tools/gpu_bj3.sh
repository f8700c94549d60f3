set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rsvd.py tests/test_gpu_id_cur.py -x -q > gpurun_out/pytest_part.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_part.log
run_exp() {  # name, env...
  env "${@:2}" timeout 500 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1; grep "sweeps" gpurun_out/exp_$1.err | sort | uniq -c | head -5
}
run_exp cross RFGPU_DEBUG=1
run_exp full RFGPU_JACOBI_CROSS=0 RFGPU_DEBUG=1
for w in c4 c2 c1; do
  for cr in 1 0; do
  RFGPU_JACOBI_CROSS=$cr RFGPU_DEBUG=1 timeout 500 python bench.py --workload $w --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$w.json 2>gpurun_out/exp_$w.err; echo "$w exit $?"
  python -c "import json; d=json.loads(open('gpurun_out/exp_$w.json').read().strip().splitlines()[-1]); print('$w cross=$cr', round(d['value']*1e3,2), {k: round(v,2) for k,v in d['phase_ms_per_step'].items() if k in ('jacobi','small_svd','single_pass_core')})"
  grep "sweeps" gpurun_out/exp_$w.err | sort | uniq -c | head -4
  done
done
