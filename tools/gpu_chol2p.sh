# Two pivots per barrier in the single-CTA Cholesky: parity, then C3 / C2 / C1 timings.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rsvd.py -x -q > gpurun_out/pytest_chol2p.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_chol2p.log
run_exp() {  # name, workload
  timeout 400 python bench.py --workload $2 --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp c3 c3
run_exp c2 c2
run_exp c1 c1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:chol_kernel -c 4 --csv python bench.py --no-e2e --no-cpu-baseline --steps 1 --warmup 0 > gpurun_out/ncu_chol2p.csv 2>gpurun_out/ncu_chol2p.err; echo "ncu exit $?"
grep -o '"gpu__time_duration.sum","[^"]*","[^"]*"' gpurun_out/ncu_chol2p.csv
