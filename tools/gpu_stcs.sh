# Slicer digit stores: plain vs streaming (__stcs) hint; the second build happens on the box.
set -x
mkdir -p gpurun_out
NCU="ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none -k regex:slice_at -c 1 --csv"
$NCU python bench.py --no-e2e --no-cpu-baseline --steps 1 --warmup 0 > gpurun_out/ncu_plain.csv 2>/dev/null; echo "ncu plain exit $?"
grep -o '"gpu__time_duration.sum","[^"]*","[^"]*"' gpurun_out/ncu_plain.csv
timeout 400 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_plain.json 2>/dev/null; python tools/exp_line.py plain
touch paper_1607_01649_b200/csrc/ozaki.cu
make -C paper_1607_01649_b200 EXTRA=-DRFGPU_SLICE_STCS > gpurun_out/make_stcs.log 2>&1; echo "make exit $?"
$NCU python bench.py --no-e2e --no-cpu-baseline --steps 1 --warmup 0 > gpurun_out/ncu_stcs.csv 2>/dev/null; echo "ncu stcs exit $?"
grep -o '"gpu__time_duration.sum","[^"]*","[^"]*"' gpurun_out/ncu_stcs.csv
timeout 400 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_stcs.json 2>/dev/null; python tools/exp_line.py stcs
timeout 400 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_stcs2.json 2>/dev/null; python tools/exp_line.py stcs2
