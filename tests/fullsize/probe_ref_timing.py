"""Reference rsvd (compiled reference, oracle/_ref) wall time on row samples of the config-3 workload, for
the CPU-baseline extrapolation: python tests/fullsize/probe_ref_timing.py ROWS[,ROWS..] THREADS[,THREADS..] OUT.json"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from oracle.oracle import get  # noqa: E402

rows_list = [int(x) for x in sys.argv[1].split(",")]
threads_list = [int(x) for x in sys.argv[2].split(",")]
ref = get("reference")
w = bench.WORKLOADS["c3"]
out = {"nproc": os.cpu_count(), "points": []}
for rows in rows_list:
    a = bench.cpu_sample_matrix(w, rows)
    for th in threads_list:
        ref.set_threads(th)
        t0 = time.perf_counter()
        ref.rsvd(a, w["k"], w["p"], w["q"], 1, False, True)
        t = time.perf_counter() - t0
        out["points"].append({"rows": rows, "threads": th, "s": t})
        print(rows, th, round(t, 3), flush=True)
        json.dump(out, open(sys.argv[3], "w"), indent=1)
