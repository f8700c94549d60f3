timeout 900 python -m pytest tests/test_gpu_rsvd.py tests/test_gpu_id_cur.py -x -q 2>&1 | tail -2
for w in c3 c2 c1; do RFGPU_JACOBI_TRACE=1 timeout 900 python bench.py --workload $w --steps 1 --warmup 0 --no-e2e --no-cpu-baseline 2>&1 | grep "jacobi c=" | head -1; done
for w in c3 c2 c1; do timeout 900 python bench.py --workload $w --no-e2e --no-cpu-baseline --steps 3 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['config']['workload'][:3], round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms_per_step'].items() if v})"; done
