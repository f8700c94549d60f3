# Single-CTA Cholesky thread count (kernel time by ncu, C1 / C3 step times).
set -x
mkdir -p gpurun_out
for t in 1024 512 256 128; do
  RFGPU_CHOL_THREADS=$t timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:chol_kernel -c 2 --csv python bench.py --no-e2e --no-cpu-baseline --steps 1 --warmup 0 > gpurun_out/ncu_cholthr_$t.csv 2>/dev/null; echo "c3 t=$t exit $?"
  grep -o '"gpu__time_duration.sum","[^"]*","[^"]*"' gpurun_out/ncu_cholthr_$t.csv | tail -1
  RFGPU_CHOL_THREADS=$t timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:chol_kernel -c 2 --csv python bench.py --workload c1 --no-e2e --no-cpu-baseline --steps 1 --warmup 0 > gpurun_out/ncu_cholthr1_$t.csv 2>/dev/null; echo "c1 t=$t exit $?"
  grep -o '"gpu__time_duration.sum","[^"]*","[^"]*"' gpurun_out/ncu_cholthr1_$t.csv | tail -1
done
RFGPU_CHOL_THREADS=256 timeout 900 python -m pytest tests/test_gpu_rsvd.py -x -q > gpurun_out/pytest_cholthr.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/pytest_cholthr.log
