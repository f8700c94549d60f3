# cp.async slicer vs the register-prefetch slicer: parity tests, then A/B at config 3 (+ ncu of both slicers).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_rsvd.py -x -q > gpurun_out/pytest_sla.log 2>&1; echo "pytest exit $?"
tail -2 gpurun_out/pytest_sla.log
run_exp() {  # name, env...
  env "${@:2}" timeout 400 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/exp_$1.json 2>gpurun_out/exp_$1.err
  echo "$1 exit $?"; python tools/exp_line.py $1
}
run_exp async
run_exp regs RFGPU_OZAKI_SLICE_ASYNC=0
run_exp async2
run_exp regs2 RFGPU_OZAKI_SLICE_ASYNC=0
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:slice_at -c 2 --csv python bench.py --no-e2e --no-cpu-baseline --steps 1 --warmup 0 > gpurun_out/ncu_sla.csv 2>gpurun_out/ncu_sla.err; echo "ncu exit $?"
RFGPU_OZAKI_SLICE_ASYNC=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:slice_at -c 2 --csv python bench.py --no-e2e --no-cpu-baseline --steps 1 --warmup 0 > gpurun_out/ncu_slr.csv 2>gpurun_out/ncu_slr.err; echo "ncu exit $?"
python -c "
import csv
for f in ['gpurun_out/ncu_sla.csv','gpurun_out/ncu_slr.csv']:
    rows=[r for r in csv.reader(open(f)) if len(r)>5]
    h=rows[0]; ik=h.index('Kernel Name'); im=h.index('Metric Name'); iv=h.index('Metric Value'); iu=h.index('Metric Unit')
    for r in rows[1:]:
        print(f[-7:-4], r[ik][:40], r[im], r[iv], r[iu])
"
