set -x
mkdir -p gpurun_out
timeout 900 python tools/pass_sweep.py > gpurun_out/pass_sweep.txt 2>&1; echo "exit $?"; cat gpurun_out/pass_sweep.txt | tail -12
