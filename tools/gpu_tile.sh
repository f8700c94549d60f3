set -x
mkdir -p gpurun_out
timeout 600 python tools/tile_overhead.py > gpurun_out/tile.txt 2>&1; echo "exit $?"
cat gpurun_out/tile.txt | tail -8
