set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -5 gpurun_out/pytest_gpu.log
run_exp() {  # name, env...
  env "${@:2}" timeout 500 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1; grep "sweeps" gpurun_out/exp_$1.err | sort | uniq -c | head -5
}
run_exp bj RFGPU_DEBUG=1
run_exp nobj RFGPU_JACOBI_BLOCK=0
for w in c4 c2 c1; do
  RFGPU_DEBUG=1 timeout 500 python bench.py --workload $w --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$w.json 2>gpurun_out/exp_$w.err; echo "$w exit $?"
  python -c "import json; d=json.loads(open('gpurun_out/exp_$w.json').read().strip().splitlines()[-1]); print('$w', d['value'], {k: round(v,2) for k,v in d['phase_ms_per_step'].items() if v})"
  grep "sweeps" gpurun_out/exp_$w.err | sort | uniq -c | head -5
done
