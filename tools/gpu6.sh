python tools/prof_small.py > gpurun_out/prof_small_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:jacobi -s 1 -c 1 -o gpurun_out/jacobi110b python tools/prof_small.py > gpurun_out/ncu_jacobi.log 2>&1
export M=4096 N=1024 K=200 P=20
python tools/prof_small.py > gpurun_out/prof_small_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:jacobi -s 1 -c 1 -o gpurun_out/jacobi220 python tools/prof_small.py > gpurun_out/ncu_jacobi2.log 2>&1
tail -n 3 gpurun_out/ncu_jacobi.log gpurun_out/ncu_jacobi2.log
