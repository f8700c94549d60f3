for w in c5 c4; do RFGPU_DEBUG=1 timeout 900 python bench.py --workload $w --no-e2e --no-cpu-baseline --steps 2 --warmup 1 2>&1 | grep -v "^\[rfgpu\] small" | tail -4; done
