"""Per-step device times of one bench workload (bench.py reports the mean): python tools/step_times.py c4 [steps].
Used to look for per-call hiccups (allocator pool growth, host round trips) behind box-to-box variance."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1607_01649_b200 as rf  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
w = bench.WORKLOADS[wl]
m, n, k, p, q = w["m"], w["n"], w["k"], w["p"], w["q"]
ell = k + p
dev = torch.device("cuda", 0)
L = rf.lib()
ctx = rf.Context(0)
At = bench.gen_shard(torch, None, w, 0, m, dev)
A = rf.DeviceMatrix.wrap(ctx, At.data_ptr(), m, n, m, f32=bool(w.get("f32")), keep=At)
Ud = torch.empty(m * ell, device=dev, dtype=torch.float64)
Dd = torch.empty(ell, device=dev, dtype=torch.float64)
Vd = torch.empty(n * ell, device=dev, dtype=torch.float64)
rank_out = C.c_int64()


def gauss(tag, r, c):
    return torch.from_numpy(rf.gaussian(bench.SEED, tag, r, c).reshape(-1, order="F")).to(dev)


if w["kind"] == "single_pass":
    Gc, Gr = gauss("spsvd.Gc", n, ell), gauss("spsvd.Gr", m, ell)

    def step():
        rf._check(L.rfgpu_single_pass_svd_device(ctx.handle, A.handle, C.c_void_p(Gc.data_ptr()), C.c_void_p(Gr.data_ptr()),
                                                 k, ell, C.c_void_p(Ud.data_ptr()), C.c_void_p(Dd.data_ptr()),
                                                 C.c_void_p(Vd.data_ptr()), C.byref(rank_out)))
else:
    G = gauss("range.G", n, ell)

    def step():
        rf._check(L.rfgpu_rsvd_device(ctx.handle, A.handle, C.c_void_p(G.data_ptr()), k, ell, q, 0,
                                      1 if w.get("reorth", True) else 0, C.c_void_p(Ud.data_ptr()),
                                      C.c_void_p(Dd.data_ptr()), C.c_void_p(Vd.data_ptr()), C.byref(rank_out)))

stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
out = []
for i in range(steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    step()
    e1.record(stream)
    e1.synchronize()
    out.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
print(wl, " ".join(f"{d:.1f}/{h:.1f}" for d, h in out), "(device ms / host wall ms per step)", flush=True)
