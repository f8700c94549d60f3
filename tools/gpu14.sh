timeout 900 python bench.py --workload c5 --no-e2e --no-cpu-baseline --steps 3 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['ms_per_step'], {k: round(v,3) for k,v in d['phase_ms_per_step'].items() if v})"
