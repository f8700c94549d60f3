"""Per-tile fixed cost of the digit GEMM: time A X and A^T Q at fixed m, l and
varying K, fit t_tile(K) = a K + b (experiment; prints one line per K)."""
import os
import sys

os.environ.setdefault("RFGPU_OZAKI", "1")
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_01649_b200 as rf

ctx = rf.Context()
m, l = 262144, 220
rows = []
for n in (1024, 2048, 4096, 8192):
    At = torch.randn(n, m, device="cuda", dtype=torch.float64)  # column-major m x n
    A = rf.DeviceMatrix.wrap(ctx, At.data_ptr(), m, n, m, keep=At)
    x = np.random.default_rng(0).standard_normal((n, l))
    q = np.random.default_rng(1).standard_normal((m, l))
    res = {}
    for trans, xx, name in ((False, x, "pass_nn"), (True, q, "pass_tn")):
        rf.multiply(A, xx, trans=trans, ctx=ctx)
        ctx.profile(True)
        ctx.profile_reset()
        for _ in range(3):
            rf.multiply(A, xx, trans=trans, ctx=ctx)
        res[name] = ctx.profile_read(name)[1] / 3
        ctx.profile(False)
    tiles_nn = (m // 128) * 4
    tiles_tn = (n // 128) * 4 * (m // 16384)
    print(f"n={n} nn {res['pass_nn']:.3f} ms ({res['pass_nn'] / (tiles_nn / 148) * 1e3:.1f} us/tile-wave, K={n}) "
          f"tn {res['pass_tn']:.3f} ms ({res['pass_tn'] / (tiles_tn / 148) * 1e3:.1f} us/tile-wave, K=16384)", flush=True)
    rows.append((n, res["pass_nn"] / (tiles_nn / 148) * 1e3))
    del A, At
    torch.cuda.empty_cache()
k = np.array([r[0] for r in rows], float)
t = np.array([r[1] for r in rows])
a, b = np.polyfit(k, t, 1)
print(f"A X per-tile time = {a * 1e3:.3f} us per 1000 K + {b:.2f} us fixed")
