"""rfgpu_rsvd_host at config-3 size from pageable vs pinned host memory under the current RFGPU_* env."""
import ctypes as C, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_1607_01649_b200 as rf
w = bench.WORKLOADS["c3"]
m, n, k, ell, q = w["m"], w["n"], w["k"], w["k"] + w["p"], w["q"]
At = bench.gen_shard(torch, None, w, 0, m, torch.device("cuda"))
Ap = np.empty((n, m)); Ap[...] = At.cpu().numpy(); del At; torch.cuda.empty_cache()
ctx = rf.Context(0); L = rf.lib()
g = rf.gaussian(1, "range.G", n, ell).reshape(-1, order="F")
U, D, V, r = np.zeros(m * ell), np.zeros(ell), np.zeros(n * ell), C.c_int64()
def call():
    rf._check(L.rfgpu_rsvd_host(ctx.handle, rf._dp(Ap.reshape(-1)), m, n, m, rf._dp(g), k, ell, q, 0, 1, rf._dp(U), rf._dp(D), rf._dp(V), C.byref(r)))
call(); call()
t0 = time.perf_counter()
for _ in range(3): call()
env = " ".join(f"{a}={b}" for a, b in sorted(os.environ.items()) if a.startswith("RFGPU_STAGE"))
print(f"[{env or 'default'}] pageable e2e {(time.perf_counter() - t0) / 3:.3f} s", flush=True)
