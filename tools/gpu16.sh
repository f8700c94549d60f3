timeout 900 python -m pytest tests/test_gpu_id_cur.py -x -q 2>&1 | tail -2
bash tools/gpu14.sh
