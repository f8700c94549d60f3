# C4 step: where the time outside the timed phases goes (sp_total / sp_alloc scopes).
mkdir -p gpurun_out
for i in 1 2; do
  timeout 600 python bench.py --workload c4 --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/c4gap_$i.json 2> gpurun_out/c4gap_$i.err; echo "c4 run $i exit $?"
  python -c "
import json; d=json.loads(open('gpurun_out/c4gap_$i.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],2), d['clocks']); print({k:round(v,2) for k,v in d['phase_ms_per_step'].items() if v})"
done
