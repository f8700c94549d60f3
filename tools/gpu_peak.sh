set -x
mkdir -p gpurun_out
(nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 500 > gpurun_out/i8peak_clocks.csv 2>&1 &) 
./tools/microbench/i8peak > gpurun_out/i8peak.txt 2>&1; echo "exit $?"
cat gpurun_out/i8peak.txt
sleep 1; tail -5 gpurun_out/i8peak_clocks.csv
