RFGPU_DEBUG=1 timeout 300 python bench.py --workload c1 --no-e2e --no-cpu-baseline --steps 1 --warmup 0 2>&1 | grep rfgpu | sort | uniq -c
RFGPU_DEBUG=1 timeout 300 python bench.py --workload c2 --no-e2e --no-cpu-baseline --steps 1 --warmup 0 2>&1 | grep rfgpu | sort | uniq -c
RFGPU_DEBUG=1 timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 1 --warmup 0 2>&1 | grep rfgpu | sort | uniq -c
