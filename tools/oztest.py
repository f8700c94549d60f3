import os, sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_1607_01649_b200 as rf
from oracle.oracle import get
port = get("port")
ctx = rf.Context(0)
for (m, n, k, p, seed) in [(600, 400, 20, 10, 1), (3000, 1000, 50, 10, 2), (20000, 3000, 100, 20, 3)]:
    sig = np.arange(1, min(m, n) + 1, dtype=np.float64) ** -1.5
    a = np.asfortranarray(port.planted(m, n, sig, seed))
    want = port.rsvd(a, k, p, 1, 5, False, True) if m * n < 5e6 else None
    res = {}
    for oz in ("0", "1"):
        os.environ["RFGPU_OZAKI"] = oz
        dm = ctx.matrix(a)
        f = rf.rsvd(dm, k, p, 1, 5, reorthonormalize=True, ctx=ctx)
        dm.free()
        res[oz] = f
    d = np.max(np.abs(res["1"].D - res["0"].D) / res["0"].D)
    w = np.max(np.abs(res["1"].D - want.D) / want.D) if want is not None else float("nan")
    sgn = np.sign(np.sum(res["1"].U * res["0"].U, axis=0))
    du = np.abs(res["1"].U * sgn - res["0"].U).max()
    print(f"m={m} n={n} k={k}: ozaki vs dmma D {d:.2e}, U {du:.2e}; ozaki vs oracle D {w:.2e}", flush=True)
