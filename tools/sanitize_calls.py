"""Smoke-size calls of every device path for compute-sanitizer (tools/sanitize_smoke.sh): rsvd on the DMMA
and INT8-digit passes (both orth modes), range finder, randomized ID / CUR, column ID, single pass (device
and streamed), svd_dense, lowrank error."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_01649_b200 as rf  # noqa: E402
from paper_1607_01649_b200 import planted as pl  # noqa: E402

ctx = rf.Context(0)
a = pl.planted_matrix(700, 500, pl.spectrum("pow2", 300), 1, noise=1e-9).numpy().T.copy(order="F")
for oz in ("0", "1"):
    os.environ["RFGPU_OZAKI"] = oz
    for reorth in (True, False):
        f = rf.rsvd(a, 20, 10, 1, 1, reorthonormalize=reorth, ctx=ctx)
    rf.rsvd(np.asfortranarray(a), 20, 10, 1, 1, reorthonormalize=True, ctx=ctx)
    rf.power_range(a, 20, 10, 1, 1, True, ctx=ctx)
    rf.randomized_id(a, 20, 10, 1, 1, ctx=ctx)
    rf.randomized_cur(a, 20, 10, 0, 1, ctx=ctx)
    rf.single_pass_svd(rf.MatrixStream(a, 64), 20, 10, 1, ctx=ctx)
rf.id_deterministic(rf.row_sketch(a, 30, 1, ctx=ctx), 20, ctx=ctx)
rf.svd_dense(a[:, :200], ctx=ctx)
print("sanitize calls done", flush=True)
