for rows in 16 32 64; do for w in c3 c2 c1; do echo -n "ROWS=$rows "; RFGPU_JACOBI_ROWS=$rows timeout 900 python bench.py --workload $w --no-e2e --no-cpu-baseline --steps 3 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['config']['workload'][:3], round(d['ms_per_step'],3), 'jacobi', round(d['phase_ms_per_step']['jacobi'],3))"; done; done
