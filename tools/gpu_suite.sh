set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_suite.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_suite.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_suite.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke_suite.log
