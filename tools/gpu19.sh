for w in c3 c2 c1; do RFGPU_JACOBI_TRACE=1 timeout 900 python bench.py --workload $w --steps 1 --warmup 0 --no-e2e --no-cpu-baseline 2>&1 | grep "jacobi c=" | head -1; done
