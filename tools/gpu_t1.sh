set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py -x -q -k single_pass > gpurun_out/pytest_t1.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_t1.log
