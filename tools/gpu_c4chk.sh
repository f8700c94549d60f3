# C4 / C3 step time with the clock sampler started before the warm-up.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=timestamp,clocks.sm --format=csv,noheader
for i in 1 2; do
timeout 600 python bench.py --workload c4 --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/exp_c4chk$i.json 2>gpurun_out/exp_c4chk$i.err; echo "exit $?"
python tools/exp_line.py c4chk$i
done
timeout 600 python bench.py --workload c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/exp_c4one.json 2>gpurun_out/exp_c4one.err; echo "exit $?"
python tools/exp_line.py c4one
timeout 600 python bench.py --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/exp_c3chk.json 2>gpurun_out/exp_c3chk.err; echo "exit $?"
python tools/exp_line.py c3chk
