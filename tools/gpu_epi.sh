# Eight epilogue warps + int64 group combination: parity, per-tile fixed cost, config 3.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_rsvd.py -x -q > gpurun_out/pytest_epi.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_epi.log
timeout 600 python tools/tile_overhead.py > gpurun_out/tile_epi.txt 2>&1; echo "tile exit $?"
tail -5 gpurun_out/tile_epi.txt
run_exp() {  # name, env...
  env "${@:2}" timeout 400 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp epi1
run_exp epi2
