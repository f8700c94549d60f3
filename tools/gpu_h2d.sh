set -x
mkdir -p gpurun_out
timeout 300 python tools/h2d_bw.py > gpurun_out/h2d.txt 2>&1; echo "exit $?"; cat gpurun_out/h2d.txt
