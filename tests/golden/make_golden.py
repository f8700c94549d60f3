"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref,
compiled from /root/reference/proj/src by oracle/Makefile).

The reference ships no stored golden vectors (every fixture is
regenerated from seeds), so these are produced by running it here, once, on
small seeded inputs; the GPU box only reads the .npz files.

Run: python tests/golden/make_golden.py   (needs oracle/_ref/librfref.so)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import get  # noqa: E402


def main():
    ref = get("reference")
    out = {}
    # rng / gaussian (proj/src/rng.cpp, sketch.cpp:56-62)
    out["g_range_1"] = ref.gaussian(1, "range.G", 64, 8)
    out["g_seek_7"] = ref.gaussian(7, "g", 5, 4)
    out["g_cur_3"] = ref.gaussian(3, "cur.G", 6, 33)
    # planted matrix (diagnostics.cpp:124-136), config-1 spectrum family
    sig = 1.0 / np.arange(1, 81, dtype=np.float64) ** 2
    a = ref.planted(120, 80, sig, 1)
    out["planted_120x80"] = a
    for reorth in (0, 1):
        f = ref.rsvd(a, 10, 5, 1, 1, False, bool(reorth))
        out[f"rsvd_r{reorth}_U"], out[f"rsvd_r{reorth}_D"], out[f"rsvd_r{reorth}_V"] = f.U, f.D, f.V
    rb = ref.power_range(a, 10, 5, 1, 1, reorth=True)
    out["range_Q"], out["range_B"], out["range_resid"] = rb.Q, rb.B, np.array([rb.residual_frob])
    # column ID / CUR (lowrank.cpp:51-70, 348-372), config-5 spectrum family
    sig5 = 10.0 ** (-6.0 * np.arange(50) / 49.0)
    a5 = ref.planted(96, 80, sig5, 1)
    out["planted_96x80"] = a5
    g = ref.gaussian(1, "cur.G", 25, 96)
    y = ref.multiply(g, a5)
    js, z, tr = ref.id_col(y, 20)
    out["cur_Y"], out["cur_Js"], out["cur_Z"] = y, js, z
    cur = ref.randomized_cur(a5, 20, 5, 0, 1)
    out["cur_full_Js"], out["cur_full_Is"], out["cur_full_U"] = cur.Js, cur.Is, cur.U
    out["cur_full_cond"] = np.array([cur.cond_C, cur.cond_R])
    is_, x, _ = ref.randomized_id(a5, 20, 5, 1, 1)
    out["rid_Is"], out["rid_X"] = is_, x
    # single pass (lowrank.cpp:160-220) at small k, stream block 7
    sig4 = np.exp(-np.arange(1, 31) / 5.0)
    a4 = ref.planted(60, 50, sig4, 1)
    out["planted_60x50"] = a4
    sp = ref.single_pass_svd(a4, 4, 4, 1, block=7)
    out["sp_U"], out["sp_D"], out["sp_V"] = sp.U, sp.D, sp.V
    path = os.path.join(HERE, "reference_fixtures.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
