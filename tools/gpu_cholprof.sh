set -x
mkdir -p gpurun_out
export M=20000 N=4000 K=200 P=20
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"chol|trinv" --csv --log-file gpurun_out/chol_launches.csv python tools/prof_small.py > gpurun_out/chol_l.log 2>&1; echo "exit $?"
timeout 600 python -m pytest tests/test_gpu_rsvd.py tests/test_gpu_ozaki.py -x -q > gpurun_out/pytest_part.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_part.log
