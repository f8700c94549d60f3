"""Profile driver: one rsvd on a config-2-family matrix (l = 110: single-CTA
Jacobi, CholeskyQR2 on 2000 x 110) for ncu captures of the small kernels."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_01649_b200 as rf  # noqa: E402

m, n = int(os.environ.get("M", 2000)), int(os.environ.get("N", 1000))
k, p = int(os.environ.get("K", 100)), int(os.environ.get("P", 10))
rng = np.random.default_rng(0)
u, _ = np.linalg.qr(rng.standard_normal((m, 500)))
v, _ = np.linalg.qr(rng.standard_normal((n, 500)))
a = np.asfortranarray((u * np.exp(-np.arange(1, 501) / 20.0)) @ v.T)
ctx = rf.Context(0)
dm = ctx.matrix(a)
for _ in range(2):
    f = rf.rsvd(dm, k, p, 2, 1, reorthonormalize=True, ctx=ctx)
print("ok", f.D[:3])
