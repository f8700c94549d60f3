set -x
mkdir -p gpurun_out
run_exp() {  # name, env...
  env "${@:2}" timeout 500 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp gap
run_exp gap2
