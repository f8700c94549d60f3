# Round-1 closing set: parity suite, smoke, bench lines for C3 (full contract) and C4 / C5 / C2 / C1.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_final.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_final.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_final.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_final_c3.json 2> gpurun_out/bench_final_c3.err; echo "bench c3 exit $?"
for w in c4 c5 c2 c1; do
  timeout 600 python bench.py --workload $w --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_final_$w.json 2> gpurun_out/bench_final_$w.err; echo "bench $w exit $?"
done
for w in c3 c4 c5 c2 c1; do python -c "
import json; d=json.loads(open('gpurun_out/bench_final_$w.json').read().strip().splitlines()[-1]); print('$w', round(d['ms_per_step'],2), round(d['roofline']['frac'],3) if d.get('roofline') else None, (d.get('e2e') or {}).get('value'), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; done
