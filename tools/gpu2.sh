free -g | head -2
nproc
timeout 300 python bench.py --workload c1 --no-e2e --no-cpu-baseline 2>&1 | tail -3
timeout 300 python bench.py --workload c2 --no-e2e --no-cpu-baseline 2>&1 | tail -3
timeout 600 python bench.py 2>&1 | tail -5
