# Host rsvd: lift panels read back on the copy stream. Parity tests + e2e.
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_rsvd.py -x -q > gpurun_out/pytest_lift.log 2>&1; echo "pytest exit $?"
tail -2 gpurun_out/pytest_lift.log
for i in 1 2; do
RFGPU_BENCH_E2E_PHASES=1 timeout 600 python bench.py --steps 3 --no-cpu-baseline > gpurun_out/exp_e2e$i.json 2> gpurun_out/exp_e2e$i.err; echo "exit $?"
grep e2e_wall gpurun_out/exp_e2e$i.err
python -c "
import json; d=json.loads(open('gpurun_out/exp_e2e$i.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'], d['clocks'])"
done
