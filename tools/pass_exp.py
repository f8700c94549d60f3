"""Config-3 passes (A X and A^T Q on the INT8 digit path, m=1048576, n=4096, l=220) timed alone: mean ms over 5
calls each, TOPS of the 28 digit products (l unpadded). This is the harness behind
profiles/r02_pass_experiments.txt: each experiment there was a temporary RFGPU_OZAKI_* switch in csrc/ozaki.cu
(printed in the line's prefix), run against the default in the same gpurun call and removed afterwards."""
import os
import sys

os.environ.setdefault("RFGPU_OZAKI", "1")
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_01649_b200 as rf

m, n, l = int(os.environ.get("PX_M", 1048576)), int(os.environ.get("PX_N", 4096)), int(os.environ.get("PX_L", 220))
ctx = rf.Context()
At = torch.randn(n, m, device="cuda", dtype=torch.float64)
A = rf.DeviceMatrix.wrap(ctx, At.data_ptr(), m, n, m, keep=At)
out = {}
for trans, rows, name in ((False, n, "pass_nn"), (True, m, "pass_tn")):
    x = np.random.default_rng(0).standard_normal((rows, l))
    rf.multiply(A, x, trans=trans, ctx=ctx)
    ctx.profile(True)
    ctx.profile_reset()
    for _ in range(5):
        rf.multiply(A, x, trans=trans, ctx=ctx)
    out[name] = ctx.profile_read(name)[1] / 5
    ctx.profile(False)
ops = 28 * 2.0 * m * n * l
env = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("RFGPU_OZAKI_"))
print(f"[{env or 'default'}] " + "  ".join(f"{k} {v:.2f} ms {ops / (v * 1e-3) / 1e12:.0f} TOPS" for k, v in out.items()),
      flush=True)
