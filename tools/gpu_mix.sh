set -x
mkdir -p gpurun_out
timeout 300 ./tools/microbench/i8mix > gpurun_out/i8mix.txt 2>&1; echo "exit $?"
cat gpurun_out/i8mix.txt
