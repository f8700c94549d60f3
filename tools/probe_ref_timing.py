import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np
import bench
from oracle.oracle import get
ref = get("reference")
w = bench.WORKLOADS["c3"]
out = {"nproc": os.cpu_count()}
for rows in (8192, 16384, 32768):
    a = bench.cpu_sample_matrix(w, rows)
    for th in (8, os.cpu_count()):
        ref.set_threads(th)
        t0 = time.perf_counter(); ref.rsvd(a, 200, 20, 1, 1, False, True); t = time.perf_counter() - t0
        out[f"{rows}_{th}"] = t
        print(rows, th, t, flush=True)
json.dump(out, open("gpurun_out/probe_ref.json", "w"))
