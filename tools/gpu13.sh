timeout 900 python -m pytest tests/test_gpu_id_cur.py -x -q 2>&1 | tail -3
RFGPU_DEBUG=1 timeout 900 python bench.py --workload c5 --no-e2e --no-cpu-baseline --steps 3 2>&1 | grep -v "^\[rfgpu\] small" | tail -2 | cut -c1-300
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:rfgpu --csv --log-file gpurun_out/launches_r01_c3.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
wc -l gpurun_out/launches_r01_c3.csv
