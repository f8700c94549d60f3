timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
for w in c5 c4 c3; do RFGPU_DEBUG=1 timeout 900 python bench.py --workload $w --no-e2e --no-cpu-baseline --steps 3 2>&1 | grep -v "^\[rfgpu\]" | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print(d['config']['workload'][:3], 'ms', round(d['ms_per_step'],3), 'tflops', round(d['sketch_tflops'],2), {k: round(v,3) for k,v in d['phase_ms_per_step'].items() if v})
"; done
