"""INT8 tensor-core peaks on this box, measured the way MEASURED_PEAKS.json measures bf16.

MEASURED_PEAKS.json (driver-written) has HBM and bf16 only; the passes over A run on the INT8
tensor cores, so their roofline denominator has to be measured here:

  * library GEMM on random data: torch._int_mm (cuBLASLt int8 x int8 -> int32) 8192^3, best of 10
    (burst) and back to back for 4 s (sustained) -- the same procedure as the driver's bf16 figure,
    which is repeated here (torch.matmul bf16 8192^3) so the two can be related on one box;
  * raw issue rate: tools/microbench/i8peak.cu (tcgen05.mma kind::i8 M=128 N=256 K=32 back to back
    from shared memory, no global traffic) on a fixed pattern tile (the round-1 figure), on zeros
    and on cycling random tiles.

SM clock and power are sampled with nvidia-smi during every sustained leg.
Usage: python tools/i8_peaks.py out.json
"""
import json
import os
import subprocess
import sys
import threading
import time

import torch


class Sampler:
    def __init__(self):
        self.rows = []
        self.stop = False
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop:
            try:
                out = subprocess.run(
                    ["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-i", "0"],
                    capture_output=True, text=True, timeout=5).stdout.strip().split(",")
                self.rows.append((float(out[0]), float(out[1])))
            except Exception:
                pass
            time.sleep(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop = True
        self.t.join()

    def summary(self):
        if not self.rows:
            return {}
        rows = sorted(self.rows)
        clk = sorted(r[0] for r in self.rows)
        pw = sorted(r[1] for r in self.rows)
        return {"sm_mhz_median": clk[len(clk) // 2], "power_w_median": pw[len(pw) // 2], "samples": len(rows)}


def gemm_leg(fn, ops):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(10):
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    reps = int(4000.0 / best) + 1
    with Sampler() as s:
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        b.synchronize()
        total = a.elapsed_time(b)
    return {"burst": ops / best / 1e9, "sustained": ops * reps / total / 1e9, "best_ms": best, "reps": reps,
            "clocks": s.summary()}


def main():
    out = {"gpu": torch.cuda.get_device_name(0)}
    n = 8192
    g = torch.Generator(device="cuda").manual_seed(1)
    a8 = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda", generator=g)
    b8 = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda", generator=g)
    ops = 2.0 * n ** 3
    try:
        out["int8_library_gemm_random_TOPS"] = gemm_leg(lambda: torch._int_mm(a8, b8), ops)
    except Exception as e:  # noqa: BLE001
        out["int8_library_gemm_random_TOPS"] = {"error": str(e)[:200]}
    z8 = torch.zeros_like(a8)
    try:
        out["int8_library_gemm_zeros_TOPS"] = gemm_leg(lambda: torch._int_mm(z8, z8), ops)
    except Exception as e:  # noqa: BLE001
        out["int8_library_gemm_zeros_TOPS"] = {"error": str(e)[:200]}
    ab = torch.randn(n, n, dtype=torch.bfloat16, device="cuda", generator=g)
    bb = torch.randn(n, n, dtype=torch.bfloat16, device="cuda", generator=g)
    out["bf16_library_gemm_random_TFLOPS"] = gemm_leg(lambda: torch.matmul(ab, bb), ops)
    del a8, b8, z8, ab, bb
    torch.cuda.empty_cache()
    exe = "/tmp/i8peak"
    src = os.path.join(os.path.dirname(os.path.abspath(__file__)), "microbench", "i8peak.cu")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe, src], check=True)
    for mode in ("pattern", "zero", "random"):
        with Sampler() as s:
            txt = subprocess.run([exe, mode], capture_output=True, text=True).stdout
        out["i8peak_" + mode] = {"text": txt.strip().splitlines(), "clocks": s.summary()}
    json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "/dev/stdout", "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
