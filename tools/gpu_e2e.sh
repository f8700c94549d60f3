set -x
mkdir -p gpurun_out
RFGPU_BENCH_E2E_PHASES=1 timeout 600 python bench.py --steps 2 --no-cpu-baseline > gpurun_out/exp_e2e.json 2> gpurun_out/exp_e2e.err; echo "exit $?"
grep e2e_wall gpurun_out/exp_e2e.err
python -c "
import json; d=json.loads(open('gpurun_out/exp_e2e.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'], d['clocks'])"
