"""Wall time of the compiled reference rsvd on the FULL config-3 matrix (the bench's A, generated on the device
and copied to host memory) at a given host thread count: python tests/fullsize/ref_full_time.py THREADS OUT.json"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from oracle.oracle import get  # noqa: E402

threads = int(sys.argv[1])
w = bench.WORKLOADS["c3"]
at = bench.gen_shard(torch, None, w, 0, w["m"], torch.device("cuda"))
a = np.asfortranarray(at.T.cpu().numpy())
del at
torch.cuda.empty_cache()
ref = get("reference")
ref.set_threads(threads)
t0 = time.perf_counter()
f = ref.rsvd(a, w["k"], w["p"], w["q"], 1, False, True)
t = time.perf_counter() - t0
gold = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                                   "config_golden.json")))["c3"]["D"]
out = {"workload": "c3 (full)", "threads": threads, "reference_s": t, "host_cores": os.cpu_count(),
       "sigma_max_rel_vs_16_thread_run": float(np.max(np.abs(f.D - np.asarray(gold)) / np.asarray(gold)))}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out), flush=True)
