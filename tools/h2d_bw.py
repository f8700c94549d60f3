"""H2D bandwidth from pinned memory: one stream vs two / four concurrent streams, and 2D row-panel copies."""
import time
import torch

n = 4 << 30  # 4 GiB
h = torch.empty(n // 8, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n // 8, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = (n // 8) // ns
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"H2D {ns} stream(s): {n / dt / 1e9:.1f} GB/s")
# D2H
torch.cuda.synchronize()
t0 = time.perf_counter()
h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
print(f"D2H 1 stream: {n / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
