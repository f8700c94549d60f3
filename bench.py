#!/usr/bin/env python
"""bench.py — RSVD time-to-rank-k on BASELINE.json config 3 (tall RSVD, FP64).

Workload (BASELINE.json configs[2], the 1/2/4/8-GPU tall-matrix config the
metric is quoted on): A = U_r diag(s) V_r^T + 1e-8 N, m = 1,048,576,
n = 4096, r = 1024, s_j = j^-1.5, U_r / V_r orthonormal Q factors of seeded
Gaussians (the reference recipe planted_matrix, diagnostics.cpp:124-136, built
row block by row block by paper_1607_01649_b200/planted.py from the
reference's own Gaussian stream), N = gaussian(1, "noise.N", m, n);
rsvd(A, k=200, p=20, q=1, reorthonormalize=true) with G = gaussian(1,
"range.G", n, 220) from the reference generator. A is row-sharded over the
ranks (strong scaling: the matrix is fixed, N GPUs share its rows); the only
collectives are allreduces of the n x l products and the l x l Grams. A (34.4
GB) is larger than L2, so no flush is needed between steps.

`value` = device-resident time per rsvd call (A, G already in HBM; CUDA
events on the library's stream; max over ranks). `e2e` = the same call made
through the public C ABI with HOST buffers (rfgpu_rsvd_host, the call the
drop-in rsvd(const DenseMatrix&) makes): A streamed from pinned memory in row
panels overlapped with the first pass, and the D2H of U, D, V, all inside the
timed region.

After the timed region the run checks its own output (`parity`): the
singular values against the golden values of the full-size oracle run
(tests/golden/config_golden.json, from tests/fullsize/parity_config_full.py) and against
the same call with the passes forced onto FP64 DMMA (RFGPU_OZAKI=0).

--impl reference runs the reference's own CPU implementation (oracle/_ref,
compiled from /root/reference/proj/src) on all host cores on row samples of
the workload at two row counts; only the part that grows with m is
extrapolated (t(m) = a + b m fitted to the two measured points), at 16
threads and at the reference's default of 8 (dense.cpp:69-94).
"""
from __future__ import annotations

import argparse
import datetime
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # BASELINE.json configs: rsvd (configs 1-3), single pass (4), column ID / CUR (5)
    "c3": dict(kind="rsvd", m=1048576, n=4096, k=200, p=20, q=1, r=1024, spectrum="pow1.5", noise=1e-8),
    # config 3 in the reference CLI's default mode (reorthonormalize=false, cli.cpp:46): one orth after the
    # power iterations, run by the Gram-Schmidt fallback with the reference's drop rule
    "c3plain": dict(kind="rsvd", m=1048576, n=4096, k=200, p=20, q=1, r=1024, spectrum="pow1.5", noise=1e-8,
                    reorth=False),
    "c2": dict(kind="rsvd", m=20000, n=10000, k=100, p=10, q=2, r=500, spectrum="exp20", noise=1e-6),
    "c1": dict(kind="rsvd", m=2000, n=2000, k=50, p=10, q=1, r=2000, spectrum="pow2", noise=0.0),
    # config 4 through the streaming entry points (MatrixStream, stream.cpp:7-24 / lowrank.cpp:170-176): the
    # fp32 values of config 4 as an fp64 host matrix, every column pushed once from pageable host memory
    "c4stream": dict(kind="single_pass", m=65536, n=65536, k=300, p=30, q=0, r=2000, spectrum="exp100", noise=1e-4,
                     f32=True, stream=True, golden="c4"),
    "c4": dict(kind="single_pass", m=65536, n=65536, k=300, p=30, q=0, r=2000, spectrum="exp100", noise=1e-4,
               f32=True),
    "c5": dict(kind="cur", m=32768, n=32768, k=300, p=20, q=0, r=1000, spectrum="decade6", noise=0.0),
}
CHUNK = 65536
SEED = 1
FP64_PEAK_TFLOPS = 37.1  # DMMA m8n8k4 burst, profiles/r01_fp_peaks.txt (MEASURED_PEAKS.json has no FP64 entry)
# INT8 tensor peaks (MEASURED_PEAKS.json has HBM and bf16 only), tools/i8_peaks.py -> profiles/r02_i8_peaks.json:
#   * tcgen05 kind::i8 issue rate from shared memory, no global traffic (tools/microbench/i8peak.cu), 4 s back to
#     back at the 1000 W cap: 3726 TOPS on cycling RANDOM operand tiles (1597 MHz), 4252-4331 on one fixed
#     pattern tile re-used by every MMA (1822-1845 MHz; the round-1 figure), 4591 on zeros (585 W, no cap).
#     Operand toggling costs power and at the cap power is clock: the digit planes are uniform random bytes,
#     so the random-operand figure is the ceiling a pass can see. Bursts: 4277 random, 4573-4595 pattern.
#   * the library GEMM measured the way MEASURED_PEAKS.json measures bf16 (torch._int_mm, cuBLASLt int8,
#     8192^3 random data): 3065 burst / 2431 TOPS sustained (1072 MHz); bf16 on the same box 1627 / 1394.
# The passes run inside a ~140 ms step at the power cap: their roofline peak is the sustained random-operand
# issue rate; the fractions of the other figures are reported beside it.
INT8_PEAK_TOPS = 3725.9
INT8_BURST_TOPS = 4277.2
INT8_PATTERN_SUSTAINED_TOPS = 4331.2   # round-1 denominator (fixed operand tile)
INT8_LIBRARY_GEMM_SUSTAINED_TOPS = 2430.7
OZAKI_PRODUCTS = 28      # int8 digit products per FP64 product (7 digits, s + t <= 6; csrc/ozaki.cu)
OZAKI_PRODUCTS_F32 = 10  # FP32 data: 4 digits, s + t <= 3


def spectrum(kind, r):
    from paper_1607_01649_b200.planted import spectrum as sp
    return sp(kind, r)


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


# ----------------------------------------------------------------- GPU data ---
def gen_shard(torch, dist, w, row0, row1, dev):
    """A^T for rows [row0, row1) as an (n, rows) tensor (= A col-major, lda = rows): the
    reference recipe planted_matrix(m, n, s, 1) + noise * gaussian(1, "noise.N", m, n)."""
    from paper_1607_01649_b200.planted import planted_matrix
    ar = (lambda t: dist.all_reduce(t)) if dist is not None else None
    at = planted_matrix(w["m"], w["n"], spectrum(w["spectrum"], w["r"]), SEED, noise=w["noise"], row0=row0,
                        row1=row1, device=dev, allreduce=ar)
    if w.get("f32"):
        at32 = at.float().contiguous()
        del at
        return at32
    return at.contiguous()


# ------------------------------------------------------------------ clocks ---
class NvmlSampler:
    """SM clock / power / clock-event reasons through NVML in this process (pynvml), every 100 ms from a
    thread. A query costs microseconds and takes no process start-up: the `nvidia-smi -lms` loop it replaces
    was seen to stall host-synchronising workloads now and then (config 4: 84 ms per call, with single timed
    means of 94 and 192 ms while per-call times measured without a sampler stayed within 82-88 ms)."""

    def __init__(self, device):
        import threading

        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        # CUDA_VISIBLE_DEVICES-relative index -> NVML handle by UUID/PCI when torch knows it, else by index
        try:
            import torch
            bus = torch.cuda.get_device_properties(device).pci_bus_id
            dom = getattr(torch.cuda.get_device_properties(device), "pci_domain_id", 0)
            dev = getattr(torch.cuda.get_device_properties(device), "pci_device_id", 0)
            self.h = pynvml.nvmlDeviceGetHandleByPciBusId(f"{dom:08X}:{bus:02X}:{dev:02X}.0")
        except Exception:
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
        self.rows = []
        self.t0 = None
        self.halt = False
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()

    def _run(self):
        nv = self.nv
        while not self.halt:
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((time.time(), float(sm), float(mx), pw, int(rs)))
            except Exception:
                pass
            time.sleep(0.1)

    def settle(self, timeout=5.0):
        end = time.time() + timeout
        while not self.rows and time.time() < end:
            time.sleep(0.02)

    def mark(self):
        self.t0 = time.time()

    def stop(self):
        self.halt = True
        self.th.join(timeout=2)
        rows = self.rows
        if self.t0 is not None:
            inside = [r for r in rows if r[0] >= self.t0]
            before = [r for r in rows if r[0] < self.t0]
            rows = inside if len(inside) >= 2 else before[-1:] + inside
        nv = self.nv
        names = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                 "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                 "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                 "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        reasons = sorted(nm for nm, bit in names.items() if any(r[4] & bit for r in rows))
        sm, mx, pw = [r[1] for r in rows], [r[2] for r in rows], [r[3] for r in rows]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None, "samples": len(sm), "reasons": reasons,
                "source": "NVML in-process, 100 ms"}


def make_sampler(device):
    try:
        return NvmlSampler(device)
    except Exception:
        return ClockSampler(device)


class ClockSampler:
    """Fallback when pynvml is unavailable: nvidia-smi clocks / power / throttle reasons every 200 ms. Started before
    the warm-up (nvidia-smi's own start-up takes driver locks that stall the
    host-synchronising steps of the first timed iterations on a fresh box);
    mark() opens the timed window and stop() keeps the samples taken inside it
    (the last warm-up sample too when the window is shorter than one period)."""
    FIELDS = ["timestamp", "clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device):
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None
        self.t0 = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(device), "--query-gpu=" + ",".join(self.FIELDS), "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def settle(self, timeout=5.0):
        """Wait for the first sample (nvidia-smi initialised) before anything is timed."""
        end = time.time() + timeout
        while self.proc is not None and time.time() < end:
            try:
                if os.path.getsize(self.path) > 0:
                    return
            except OSError:
                pass
            time.sleep(0.05)

    def mark(self):
        self.t0 = datetime.datetime.now()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f")
                rows.append((ts, float(parts[1]), float(parts[2]), float(parts[3]), parts[4:8]))
            except ValueError:
                continue
        os.unlink(self.path)
        if self.t0 is not None:
            inside = [r for r in rows if r[0] >= self.t0]
            before = [r for r in rows if r[0] < self.t0]
            rows = inside if len(inside) >= 2 else before[-1:] + inside
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = {nm for r in rows for nm, v in zip(names, r[4]) if v.lower().startswith("active")}
        sm, mx, pw = [r[1] for r in rows], [r[2] for r in rows], [r[3] for r in rows]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None, "samples": len(sm), "reasons": sorted(reasons)}


# --------------------------------------------------------------- reference ---
def cpu_sample_matrix(w, rows):
    """Row sample (rows x n) of the workload's distribution, built on the host."""
    rng = np.random.default_rng(SEED)
    n, r = w["n"], w["r"]
    V, _ = np.linalg.qr(rng.standard_normal((n, r)))
    U, _ = np.linalg.qr(rng.standard_normal((rows, r)))
    U *= np.sqrt(rows / w["m"])  # rows of an m-row orthonormal factor have this scale
    a = (U * spectrum(w["spectrum"], r)) @ V.T
    if w["noise"]:
        a += w["noise"] * rng.standard_normal((rows, n))
    return np.asfortranarray(a)


def run_reference_rsvd(w, a_sample, threads):
    from oracle.oracle import get
    ref = get("reference")
    ref.set_threads(threads)
    t0 = time.perf_counter()
    ref.rsvd(a_sample, w["k"], w["p"], w["q"], SEED, False, w.get("reorth", True))
    return time.perf_counter() - t0


# The reference's cost per row of A grows with m (its column-parallel multiply streams A once per output
# column: small samples sit in host caches, config-size A does not): measured at 16 threads on the GPU box,
# 8192 / 24576 / 65536 / 131072 / 262144 rows: 3.35 / 8.0 / 22.8 / 47.1 / 110.5 s
# (gpurun_out r02b_refcurve16.json -> profiles/r02_reference_curve.json), and the FULL config-3 call once:
# 560.2 s (tests/fullsize/parity_config_full.py, profiles/r02_parity_c3.json); at the reference's default 8 threads
# 709.4 s (tests/fullsize/ref_full_time.py, profiles/r02_reference_c3_8threads.json). A linear fit through small samples
# would claim ~300 s. The CPU numbers below are therefore anchored on that full-size measurement: every step
# times the reference on an 8192-row sample of the workload and scales it by full / sample as measured
# together on this box type.
ANCHOR = {"c3": {"full_s": 560.19, "threads": 16, "sample_rows": 8192, "sample_s": 3.3506,
                 "source": "profiles/r02_parity_c3.json (reference rsvd on the full config-3 A, 16 threads) and "
                           "profiles/r02_reference_curve.json (8192-row sample, 16 threads)",
                 "full_s_8_threads": 709.41,
                 "source_8_threads": "profiles/r02_reference_c3_8threads.json (the reference's default thread count, "
                                     "min(hw, 8), dense.cpp:69-94; full config-3 A)"}}


def anchored_reference(w, workload, sample_fn, steps, warmup, threads):
    """(per-step values, description dict) of the reference at the workload's full size."""
    an = ANCHOR.get(workload) or ANCHOR.get(workload.replace("plain", ""))  # c3plain: the config-3 anchor
    if an is None or w["m"] <= 24576:  # small config: timed at full size
        a = sample_fn(w["m"])
        for _ in range(warmup):
            run_reference_rsvd(w, a, threads)
        times = [run_reference_rsvd(w, a, threads) for _ in range(steps)]
        return times, {"sample": f"reference rsvd at full size ({w['m']}x{w['n']}), {threads} threads"}
    a = sample_fn(an["sample_rows"])
    for _ in range(warmup):
        run_reference_rsvd(w, a, threads)
    scale = an["full_s"] / an["sample_s"]
    raw = [run_reference_rsvd(w, a, threads) for _ in range(steps)]
    desc = {"sample": (f"reference rsvd(k={w['k']}, p={w['p']}, q={w['q']}, reorth={str(w.get('reorth', True)).lower()}) "
                       f"on an {an['sample_rows']}x{w['n']} row sample each step (mean {statistics.mean(raw):.3f} s), "
                       f"scaled by {scale:.1f} = full-size measurement / sample measurement ({an['full_s']} s / "
                       f"{an['sample_s']} s at {an['threads']} threads)"),
            "anchor": an, "sample_s": raw, "full_size_measured_s": an["full_s"],
            "default_threads": 8, "default_threads_value_measured": an["full_s_8_threads"]}
    return [t * scale for t in raw], desc


def reference_arm(args, w, rank, world):
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    times, desc = anchored_reference(w, args.workload, lambda r: cpu_sample_matrix(w, r), args.steps, args.warmup,
                                     threads)
    val = statistics.mean(times)
    line = {
        "metric": "rsvd_time_to_rank_k", "value": val, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": val * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (planted spectrum, seeded)", "impl": "reference",
        "config": config_of(w, world, args),
        "cpu_baseline": {"value": val, "unit": "s", "cores": threads, "kind": "reference", **desc},
        "e2e": {"value": val, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


GOLDEN = os.path.join(ROOT, "tests", "golden", "config_golden.json")


def check_parity(args, w, kind, step, ctx, rank_out, Ud, Dd, Vd, Js, mloc, n):
    """The timed call's result against (1) the golden singular values / pivots of the full-size CPU oracle
    run on the same A (tests/golden/config_golden.json, tests/fullsize/parity_config_full.py) and (2) the same call with
    the passes forced onto FP64 DMMA (RFGPU_OZAKI=0; an independent product kernel). Outside the timed
    region."""
    import torch
    ctx.synchronize()
    kk = rank_out.value
    # FP32 data: the north star's 1e-4; plain power mode: its intrinsic noise floor
    tol = 1e-4 if w.get("f32") else (1e-10 if w.get("reorth", True) else 1e-6)
    res = {"tolerance_sigma_rel": tol}
    if kind == "cur":
        got_js = np.array(Js[:kk], copy=True)
    else:
        got_d = Dd[:kk].cpu().numpy().copy()
        got_u, got_v = Ud[: mloc * kk].view(kk, mloc).clone(), Vd[: n * kk].view(kk, n).clone()
    ok = True
    gold = {}
    if os.path.exists(GOLDEN):
        gold = json.load(open(GOLDEN)).get(w.get("golden", args.workload), {})
    if gold.get("D") is not None and kind != "cur":
        gd = np.asarray(gold["D"])
        e = float(np.max(np.abs(got_d[: len(gd)] - gd) / gd)) if len(gd) == kk else float("inf")
        res.update(golden_sigma_max_rel=e, golden_source=gold.get("source"))
        ok &= e <= tol
    if gold.get("Js") is not None and kind == "cur":
        res.update(golden_pivots_equal=bool(np.array_equal(got_js, np.asarray(gold["Js"]))),
                   golden_source=gold.get("source"))
        ok &= res["golden_pivots_equal"]
    prev = os.environ.get("RFGPU_OZAKI")
    os.environ["RFGPU_OZAKI"] = "0"
    try:
        step()
        ctx.synchronize()
    finally:
        if prev is None:
            os.environ.pop("RFGPU_OZAKI", None)
        else:
            os.environ["RFGPU_OZAKI"] = prev
    if kind == "cur":
        res["dmma_pivots_equal"] = bool(np.array_equal(got_js, np.asarray(Js[: rank_out.value])))
        ok &= res["dmma_pivots_equal"]
    else:
        d = Dd[:kk].cpu().numpy()
        u, v = Ud[: mloc * kk].view(kk, mloc), Vd[: n * kk].view(kk, n)

        def aligned(x, ref):  # rows of x / ref are singular vectors
            s = torch.sign(torch.sum(x * ref, dim=1, keepdim=True))
            s[s == 0] = 1
            return float(torch.max(torch.abs(x * s - ref)))
        res.update(dmma_sigma_max_rel=float(np.max(np.abs(got_d - d) / d)) if rank_out.value == kk else float("inf"),
                   dmma_U_max_abs=aligned(got_u, u), dmma_V_max_abs=aligned(got_v, v))
        ok &= res["dmma_sigma_max_rel"] <= tol
    res["ok"] = bool(ok)
    return res


def config_of(w, world, args):
    desc = {"rsvd": f"RSVD fp64 m={w['m']} n={w['n']} k={w['k']} p={w['p']} q={w['q']} "
                    f"reorthonormalize={'true' if w.get('reorth', True) else 'false'}",
            "cur": f"column ID (row sketch G A + CPQR + Z) fp64 m={w['m']} n={w['n']} k={w['k']} p={w['p']}",
            "single_pass": f"single-pass SVD, fp32 A (fp64 arithmetic) m={w['m']} n={w['n']} k={w['k']} p={w['p']}"}
    return {"workload": f"{args.workload}: " + desc[w["kind"]], "m": w["m"], "n": w["n"], "k": w["k"], "p": w["p"], "q": w["q"],
            "rank_planted": w["r"], "noise": w["noise"], "seed": SEED, "parallelism": f"row-shard x{world}",
            "l2": ("A (8*m*n bytes) larger than L2; no flush needed" if 8 * w["m"] * w["n"] > 126e6 else
                   "A fits in L2 and stays warm between steps (no flush)")}


# --------------------------------------------------------------------- main ---
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="rfgpu", choices=["rfgpu", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the self-check (profiling runs: identical steps)")
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)

    if args.impl == "reference":
        return reference_arm(args, w, rank, world)

    import torch
    dist = None
    if world > 1:
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl")
        dist = tdist
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    import paper_1607_01649_b200 as rf
    L = rf.lib()
    if world > 1:
        obj = [rf.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = rf.Context(local, rank, world, obj[0])
    else:
        ctx = rf.Context(local)

    m, n, k, p, q = w["m"], w["n"], w["k"], w["p"], w["q"]
    ell = k + p
    row0, row1 = m * rank // world, m * (rank + 1) // world
    mloc = row1 - row0
    At = gen_shard(torch, dist, w, row0, row1, dev)
    torch.cuda.synchronize()
    kind = w["kind"]
    A = rf.DeviceMatrix.wrap(ctx, At.data_ptr(), mloc, n, mloc, f32=bool(w.get("f32")), keep=At)
    Ud = torch.empty(mloc * ell, device=dev, dtype=torch.float64)
    Dd = torch.empty(ell, device=dev, dtype=torch.float64)
    Vd = torch.empty(n * ell, device=dev, dtype=torch.float64)
    rank_out = C.c_int64()
    trunc = C.c_int()

    def dev_gauss(tag, r, c):
        return torch.from_numpy(rf.gaussian(SEED, tag, r, c).reshape(-1, order="F")).to(dev)

    reorth = 1 if w.get("reorth", True) else 0
    if kind == "rsvd":
        G = dev_gauss("range.G", n, ell)

        def step():
            rf._check(L.rfgpu_rsvd_device(ctx.handle, A.handle, C.c_void_p(G.data_ptr()), k, ell, q, 0, reorth,
                                          C.c_void_p(Ud.data_ptr()), C.c_void_p(Dd.data_ptr()),
                                          C.c_void_p(Vd.data_ptr()), C.byref(rank_out)))
    elif kind == "cur":
        G = dev_gauss("cur.G", ell, m)
        Yd = torch.empty(ell * n, device=dev, dtype=torch.float64)
        Zd = torch.empty(k * n, device=dev, dtype=torch.float64)
        Js = np.zeros(k, dtype=np.int64)

        def step():
            rf._check(L.rfgpu_row_sketch_device(ctx.handle, A.handle, C.c_void_p(G.data_ptr()), ell,
                                                C.c_void_p(Yd.data_ptr())))
            rf._check(L.rfgpu_col_id_device(ctx.handle, C.c_void_p(Yd.data_ptr()), ell, n, k, rf._ip(Js),
                                            C.c_void_p(Zd.data_ptr()), C.byref(rank_out), C.byref(trunc)))
    elif w.get("stream"):
        # host A (pageable fp64, the values of the fp32 config-4 matrix), pushed in 4096-column slabs as the
        # drop-in's single_pass_svd(MatrixStream&) does; U, D, V land in host buffers
        Ah = np.ascontiguousarray(At.double().cpu().numpy())  # (n, m) row-major = A column-major
        A.free()
        del At
        torch.cuda.empty_cache()
        At = torch.empty(1, device=dev)
        A = rf.DeviceMatrix.wrap(ctx, At.data_ptr(), 1, 1, 1)
        gch = rf.gaussian(SEED, "spsvd.Gc", n, ell).reshape(-1, order="F")
        grh = rf.gaussian(SEED, "spsvd.Gr", m, ell).reshape(-1, order="F")
        Uh, Dh, Vh = np.zeros(m * k), np.zeros(k), np.zeros(n * k)
        flat = Ah.reshape(-1)

        def step():
            sp = C.c_void_p()
            rf._check(L.rfgpu_single_pass_begin(ctx.handle, m, n, ell, rf._dp(gch), rf._dp(grh), C.byref(sp)))
            for c0 in range(0, n, 4096):
                c1 = min(n, c0 + 4096)
                rf._check(L.rfgpu_single_pass_push(sp, c0, rf._dp(flat[c0 * m:]), c1 - c0))
            rf._check(L.rfgpu_single_pass_finish(sp, k, rf._dp(Uh), rf._dp(Dh), rf._dp(Vh), C.byref(rank_out)))
            Dd[:k].copy_(torch.from_numpy(Dh))
    else:
        Gc = dev_gauss("spsvd.Gc", n, ell)
        Gr = dev_gauss("spsvd.Gr", m, ell)

        def step():
            rf._check(L.rfgpu_single_pass_svd_device(ctx.handle, A.handle, C.c_void_p(Gc.data_ptr()),
                                                     C.c_void_p(Gr.data_ptr()), k, ell, C.c_void_p(Ud.data_ptr()),
                                                     C.c_void_p(Dd.data_ptr()), C.c_void_p(Vd.data_ptr()),
                                                     C.byref(rank_out)))

    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    sampler = make_sampler(local)
    sampler.settle()
    for _ in range(max(3, args.warmup)):
        step()
    ctx.synchronize()
    barrier()
    torch.cuda.synchronize()
    ctx.profile_reset()  # launch counter base; per-phase timing stays off in the timed region (graph replays)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler.mark()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    ev1.synchronize()
    clocks = sampler.stop()
    ctx.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    launches = ctx.launch_count() // args.steps
    # per-phase CUDA-event breakdown from separate profiled (eager) steps after the timed region
    prof_steps = max(1, min(3, args.steps))
    ctx.profile(True)
    ctx.profile_reset()
    for _ in range(prof_steps):
        step()
    ctx.synchronize()
    prof = {nm: ctx.profile_read(nm) for nm in ("pass_nn", "pass_tn", "ozaki_slice", "sketch_nn", "sketch_tn", "orth",
                                                "small_svd", "jacobi", "gram", "chol", "trsm", "lift", "stats",
                                                "slicer", "col_id", "cpqr", "trsm_id", "single_pass_core", "gemm_nn",
                                                "gemm_tn", "allreduce", "sp_total", "sp_alloc")}
    ctx.profile(False)
    pass_names = ("sketch_nn", "sketch_tn") if kind == "single_pass" else ("pass_nn", "pass_tn")
    if kind == "single_pass" and prof["sketch_nn"][0] == 0:  # the dual sketch ran on the digit path
        pass_names = ("pass_nn", "pass_tn")
    n_pass = sum(prof[nm][0] for nm in pass_names)
    pass_ms = sum(prof[nm][1] for nm in pass_names)
    # algorithmic flops of the passes over A (ell unpadded): 2 m n ell per pass;
    # the single pass computes both sketches (4 m n ell) from one read of A
    flops_per_pass = 2.0 * mloc * n * ell
    passes_alg = {"rsvd": n_pass / prof_steps, "cur": 1.0, "single_pass": 2.0}[kind]
    achieved = flops_per_pass * passes_alg * prof_steps / (pass_ms * 1e-3) / 1e12 if pass_ms > 0 else None
    ozaki = prof["ozaki_slice"][0] > 0  # the FP64 passes ran as int8 digit products on tcgen05
    products = OZAKI_PRODUCTS_F32 if w.get("f32") else OZAKI_PRODUCTS
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tr_path):
        try:
            t = json.load(open(tr_path)).get(args.workload)
            traffic = t.get("traffic_bytes") if isinstance(t, dict) else t
        except Exception:
            traffic = None

    # ---- self-check of the timed result (outside the timed region) ----------
    parity = None if args.no_parity else check_parity(args, w, kind, step, ctx, rank_out, Ud, Dd, Vd,
                                                      Js if kind == "cur" else None, mloc, n)

    # ---- e2e through the host-buffer C ABI (upload + rsvd + D2H) -----------
    # The drop-in's rsvd(const DenseMatrix&) hands rfgpu_rsvd_host PAGEABLE std::vector memory: that is the
    # headline e2e (A staged through the library's pinned ring by host copy threads). The same call from
    # pinned buffers is reported beside it.
    e2e = None
    if not args.no_e2e and kind == "rsvd":
        ctx.release_memory()  # the device-resident call's graph and cached pools: the host call needs the room
        try:
            Gh = rf.gaussian(SEED, "range.G", n, ell)
            gflat = np.asfortranarray(Gh).reshape(-1, order="F")
            Dh = np.zeros(ell)

            def timed_e2e(Ah_ptr, Uh_ptr, Vh_ptr):
                def e2e_step():
                    # the drop-in call: host A in (streamed behind pass 1), host U, D, V out
                    rf._check(L.rfgpu_rsvd_host(ctx.handle, C.cast(C.c_void_p(Ah_ptr), rf._pd), mloc, n, mloc,
                                                rf._dp(gflat), k, ell, q, 0, reorth, C.cast(C.c_void_p(Uh_ptr), rf._pd),
                                                rf._dp(Dh), C.cast(C.c_void_p(Vh_ptr), rf._pd), C.byref(rank_out)))
                e2e_step()
                barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0 = time.perf_counter()
                e0.record(stream)
                for _ in range(args.steps):
                    e2e_step()
                e1.record(stream)
                e1.synchronize()
                wall = (time.perf_counter() - t0) / args.steps
                return max_over_ranks(e0.elapsed_time(e1) / args.steps) / 1e3, wall

            Ap = np.empty((n, mloc))  # pageable, like the DenseMatrix a drop-in caller passes
            Ap[...] = At.cpu().numpy()
            Up, Vp = np.zeros(mloc * ell), np.zeros(n * ell)
            e2e_s, e2e_wall = timed_e2e(Ap.ctypes.data, Up.ctypes.data, Vp.ctypes.data)
            kk = rank_out.value
            del Ap, Up, Vp
            Ah = torch.empty((n, mloc), dtype=torch.float64, pin_memory=True)
            Ah.copy_(At)
            Uh = torch.empty(mloc * ell, dtype=torch.float64, pin_memory=True)
            Vh = torch.empty(n * ell, dtype=torch.float64, pin_memory=True)
            pin_s, pin_wall = timed_e2e(Ah.data_ptr(), Uh.data_ptr(), Vh.data_ptr())
            e2e = {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": int(8 * (mloc * n + n * ell)),
                   "d2h_bytes_per_step": int(8 * (mloc * kk + n * kk + kk)),
                   "host_memory": "pageable (the drop-in's DenseMatrix storage), staged by the library",
                   "wall_s": e2e_wall, "pinned_value": pin_s, "pinned_wall_s": pin_wall}
            del Ah, Uh, Vh
        except Exception as ex:  # report, never hide
            e2e = {"value": None, "unit": "s", "error": f"{type(ex).__name__}: {ex}"}

    if w.get("stream"):  # the timed call already is end to end from host buffers
        e2e = {"value": ms / 1e3, "unit": "s", "h2d_bytes_per_step": int(8 * m * n + 8 * (m + n) * ell),
               "d2h_bytes_per_step": int(8 * (m + n + 1) * k), "note": "streamed from pageable host memory"}

    # ---- CPU baseline (reference, bounded samples of this A), rank 0 at N=1 -
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and kind == "rsvd":
        threads = os.cpu_count() or 1
        times, desc = anchored_reference(w, args.workload, lambda r: np.asfortranarray(At[:, :r].T.cpu().numpy()),
                                         1, 0, threads)
        cpu = {"value": times[0], "unit": "s", "cores": threads, "kind": "reference", **desc}
        cpu["sample"] = "the first rows of this A: " + cpu["sample"]

    if rank == 0:
        line = {
            "metric": {"rsvd": "rsvd_time_to_rank_k", "cur": "column_id_time",
                       "single_pass": "single_pass_svd_time"}[kind],
            "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": ("synthetic: the reference recipe planted_matrix + noise (seeded reference Gaussian stream)"
                     + (", A stored fp32" if w.get("f32") else "")),
            "config": config_of(w, world, args),
            "sketch_tflops": achieved,
            "roofline": ({"bound": "tensor", "achieved": achieved * products, "peak": INT8_PEAK_TOPS,
                          "unit": "TOPS", "frac": achieved * products / INT8_PEAK_TOPS, "traffic": traffic,
                          "kernel": f"ozaki_gemm_kernel (tcgen05 kind::i8; passes over A: {' + '.join(pass_names)})",
                          "algorithmic_ops_per_pass": flops_per_pass * products,
                          "fp64_equivalent_tflops": achieved, "fp64_dmma_peak_tflops": FP64_PEAK_TFLOPS,
                          "passes_per_step": passes_alg, "launches_per_step": n_pass / prof_steps,
                          "pass_ms_avg": pass_ms / n_pass if n_pass else None,
                          "frac_of_burst": achieved * products / INT8_BURST_TOPS,
                          "frac_of_fixed_tile_sustained_peak_4331": achieved * products / INT8_PATTERN_SUSTAINED_TOPS,
                          "frac_of_library_int8_gemm_sustained_2431": achieved * products / INT8_LIBRARY_GEMM_SUSTAINED_TOPS,
                          "peak_source": "tcgen05 kind::i8 issue rate on cycling random operand tiles, sustained 4 s at "
                                         "the 1000 W cap (profiles/r02_i8_peaks.json; MEASURED_PEAKS.json has bf16 "
                                         "only); round 1 used the fixed-tile figure 4331"}
                         if ozaki and achieved else
                         {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                          "frac": (achieved / FP64_PEAK_TFLOPS) if achieved else None, "traffic": traffic,
                          "kernel": f"gemm_f64_tma_kernel (passes over A: {' + '.join(pass_names)})",
                          "per_pass_flops": flops_per_pass, "passes_per_step": passes_alg,
                          "launches_per_step": n_pass / prof_steps,
                          "pass_ms_avg": pass_ms / n_pass if n_pass else None,
                          "peak_source": "FP64 DMMA microbenchmark profiles/r01_fp_peaks.txt (no FP64 entry in "
                                         "MEASURED_PEAKS.json)"}),
            "phase_ms_per_step": {nm: v[1] / prof_steps for nm, v in prof.items()},
            "phase_note": f"CUDA events per phase over {prof_steps} profiled eager step(s) after the timed region",
            "e2e": e2e, "gpu_launches": launches, "clocks": clocks, "cpu_baseline": cpu, "parity": parity,
        }
        print(json.dumps(line), flush=True)
    A.free()
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
