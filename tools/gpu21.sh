timeout 1500 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -2
for w in c3 c2 c1 c4 c5; do timeout 900 python bench.py --workload $w --no-e2e --no-cpu-baseline --steps 3 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['config']['workload'][:3], round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms_per_step'].items() if v})"; done
