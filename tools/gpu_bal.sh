set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_rsvd.py -x -q > gpurun_out/pytest_part.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_part.log
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"slice|stats" --csv --log-file gpurun_out/l_bal.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu exit $?"
