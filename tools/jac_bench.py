"""Jacobi small-SVD timing sweep: svd_dense of graded l x l matrices (the
R factors the range finder hands to jacobi_svd), jacobi phase time + sweeps."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_01649_b200 as rf  # noqa: E402

ctx = rf.Context(0)
ctx.profile(True)
for ell in [int(x) for x in os.environ.get("ELLS", "60,110,220,330").split(",")]:
    rng = np.random.default_rng(ell)
    u, _ = np.linalg.qr(rng.standard_normal((4 * ell, ell)))
    v, _ = np.linalg.qr(rng.standard_normal((ell, ell)))
    a = np.asfortranarray((u * np.arange(1, ell + 1) ** -1.5) @ v.T)
    rf.svd_dense(a, ctx=ctx)
    ctx.profile_reset()
    reps = 3
    for _ in range(reps):
        f = rf.svd_dense(a, ctx=ctx)
    n, ms = ctx.profile_read("jacobi")
    s = np.linalg.svd(a, compute_uv=False)
    print(f"ell={ell} jacobi {ms / reps:.3f} ms  max rel err {np.max(np.abs(f.D[:ell] - s) / s):.2e}", flush=True)
