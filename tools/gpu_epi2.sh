# Persistent tile loop with the faster epilogue.
set -x
mkdir -p gpurun_out
RFGPU_OZAKI_PERSIST=1 timeout 600 python tools/tile_overhead.py > gpurun_out/tile_pers.txt 2>&1; echo "tile exit $?"
tail -5 gpurun_out/tile_pers.txt
run_exp() {  # name, env...
  env "${@:2}" timeout 400 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp pers RFGPU_OZAKI_PERSIST=1
run_exp base
run_exp pers2 RFGPU_OZAKI_PERSIST=1
