"""One-line summary of a bench.py experiment run (gpurun_out/exp_<name>.json)."""
import json
import sys

name = sys.argv[1]
d = json.loads(open(f"gpurun_out/exp_{name}.json").read().strip().splitlines()[-1])
ph = d["phase_ms_per_step"]
keys = ["pass_nn", "pass_tn", "ozaki_slice", "stats", "slicer", "orth", "small_svd", "jacobi", "gram", "chol", "trsm",
        "lift"]
print(name, round(d["value"] * 1e3, 2), "samples", d.get("clocks", {}).get("samples"), " ".join(f"{k}={ph[k]:.2f}" for k in keys if k in ph),
      "clk", d.get("clocks", {}).get("sm_mhz"), d.get("clocks", {}).get("reasons"))
