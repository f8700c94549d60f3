"""H2D bandwidth from pinned memory: one stream vs two / four concurrent streams (experiment)."""
import time
import torch

n = 4 << 30  # 4 GiB
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    part = n // ns
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"streams={ns}: {n / dt / 1e9:.1f} GB/s", flush=True)
torch.cuda.synchronize()
t = time.perf_counter()
h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
print(f"D2H 1 stream: {n / (time.perf_counter() - t) / 1e9:.1f} GB/s")
