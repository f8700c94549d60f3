import os, sys, numpy as np
sys.path.insert(0, "/root/repo")
os.environ["RFGPU_OZAKI"] = "1"
import paper_1607_01649_b200 as rf
ctx = rf.Context(0)
def err(a, x, trans):
    got = rf.multiply(np.asfortranarray(a), x, trans=trans, ctx=ctx)
    al, xl = a.astype(np.longdouble), x.astype(np.longdouble)
    want = al.T @ xl if trans else al @ xl
    rows = np.abs(a).max(axis=0 if trans else 1); cols = np.abs(x).max(axis=0)
    sc = np.outer(rows, cols); sc[sc == 0] = 1
    e = np.abs(got - want) / sc
    i, j = np.unravel_index(np.argmax(e), e.shape)
    return float(e.max()), (i, j)
rng = np.random.default_rng(1)
for name in ["plain", "row3big", "row5tiny", "row7zero", "col2small", "x1big", "x2zero", "all"]:
    m, n, c = 1000, 777, 40
    a = rng.standard_normal((m, n)); x = rng.standard_normal((m, c))
    if name in ("row3big", "all"): a[3] *= 1e120
    if name in ("row5tiny", "all"): a[5] *= 1e-150
    if name in ("row7zero", "all"): a[7] = 0
    if name in ("col2small", "all"): a[:, 2] *= 1e-8
    if name in ("x1big", "all"): x[:, 1] *= 1e80
    if name in ("x2zero", "all"): x[:, 2] = 0
    print(name, "TN", err(a, x, True), "NN", err(a, rng.standard_normal((n, c)), False), flush=True)
