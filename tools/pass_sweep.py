"""Digit-GEMM pass throughput over shapes (A X and A^T Q through rfgpu_multiply
on the INT8 digit path): TOPS of the 28 digit products and the fraction of the
sustained INT8 peak, per (m, n, l). Prints one line per shape."""
import os
import sys

os.environ.setdefault("RFGPU_OZAKI", "1")
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_01649_b200 as rf

PEAK = 4331.2  # TOPS, profiles/r01_i8_peak.txt (sustained)
ctx = rf.Context()
shapes = [(262144, 4096, 220), (524288, 4096, 220), (1048576, 4096, 220), (1048576, 4096, 64), (1048576, 4096, 128),
          (1048576, 4096, 320), (131072, 32768, 220), (32768, 32768, 320)]
for m, n, l in shapes:
    At = torch.randn(n, m, device="cuda", dtype=torch.float64)
    A = rf.DeviceMatrix.wrap(ctx, At.data_ptr(), m, n, m, keep=At)
    res = {}
    for trans, rows, name in ((False, n, "pass_nn"), (True, m, "pass_tn")):
        x = np.random.default_rng(0).standard_normal((rows, l))
        rf.multiply(A, x, trans=trans, ctx=ctx)
        ctx.profile(True)
        ctx.profile_reset()
        for _ in range(3):
            rf.multiply(A, x, trans=trans, ctx=ctx)
        res[name] = ctx.profile_read(name)[1] / 3
        ctx.profile(False)
    ops = 28 * 2.0 * m * n * (-(-l // 16) * 16)
    line = f"m={m} n={n} l={l}:"
    for k in ("pass_nn", "pass_tn"):
        tops = ops / (res[k] * 1e-3) / 1e12
        line += f"  {k} {res[k]:.2f} ms {tops:.0f} TOPS frac {tops / PEAK:.3f}"
    print(line, flush=True)
    del A, At
    torch.cuda.empty_cache()
