"""Summarise a gpurun profiling set into profiles/ (tracked):

  python tools/summarize_prof.py <round> <workload> [steps_in_launch_list]

reads gpurun_out/launches_<round>_<workload>.csv (ncu launch list of
`bench.py --steps 1 --warmup W`) and gpurun_out/top_<round>_<workload>.ncu-rep
(ncu --set full of the GEMM launches), writes
  profiles/<round>_launches_<workload>.csv        this library's launches of the timed step
  profiles/<round>_launches_<workload>_summary.txt per-kernel count / time / share of the step
  profiles/<round>_ncu_top_kernels_<workload>.jsonl key metrics per captured launch
  profiles/ncu_traffic.json                        DRAM bytes of the largest pass launch (bench.py roofline.traffic)
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OURS = ("gemm_f64", "jacobi_svd", "chol_inv", "trinv_upper", "cpqr", "reduce_splits", "symmetrize", "sumsq",
        "sum_array", "transpose", "gather_", "lsq_scale", "gs_", "add_inplace", "sylvester", "f32_to_f64",
        "scale_", "copy_", "fill_", "ozaki_gemm", "stats_kernel", "slice_a_kernel", "slice_r_kernel", "colexp_kernel",
        "col_exp_kernel", "rowexp_kernel", "reduce_ws_kernel", "chol_kernel", "trinv_smem", "slice_at_kernel", "slice_at_async",
        "colexp_fix", "cholb_", "rfgpu")


def ours(name):
    return not name.startswith("void at::") and "at::native" not in name and any(t in name for t in OURS)


def short(name):
    n = name.replace("void ", "").replace("<unnamed>::", "").replace("unnamed>::", "").replace("(anonymous namespace)::", "")
    return n.split("(")[0]


def launches(rnd, wl, steps_total):
    path = os.path.join(ROOT, "gpurun_out", f"launches_{rnd}_{wl}.csv")
    text = open(path).read()
    text = text[text.index('"ID"'):]
    rows = [r for r in csv.DictReader(io.StringIO(text)) if r["Metric Name"] == "gpu__time_duration.sum"]
    mine = [r for r in rows if ours(r["Kernel Name"])]
    per_step = len(mine) // steps_total
    last = mine[-per_step:]
    out_csv = os.path.join(ROOT, "profiles", f"{rnd}_launches_{wl}.csv")
    with open(out_csv, "w") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "grid", "block", "duration_ns"])
        for r in last:
            w.writerow([short(r["Kernel Name"]), r["Grid Size"], r["Block Size"], r["Metric Value"]])
    agg = defaultdict(lambda: [0, 0.0])
    for r in last:
        a = agg[short(r["Kernel Name"])]
        a[0] += 1
        a[1] += float(r["Metric Value"]) / 1e6
    tot = sum(v[1] for v in agg.values())
    lines = [f"# {rnd} {wl}: this library's launches in ONE timed step (last {per_step} of {len(mine)} launches; "
             f"ncu --metrics gpu__time_duration.sum --clock-control none: cold-cache, serialised)",
             f"# total {tot:.3f} ms over {per_step} launches", f"{'kernel':70s} {'count':>5s} {'ms':>10s} {'share':>7s}"]
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k[:70]:70s} {n:5d} {ms:10.3f} {100 * ms / tot:6.2f}%")
    open(os.path.join(ROOT, "profiles", f"{rnd}_launches_{wl}_summary.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__registers_per_thread",
           "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
           "sm__cycles_elapsed.avg.per_second", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu_full(rnd, wl):
    rep = os.path.join(ROOT, "gpurun_out", f"top_{rnd}_{wl}.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out, best, passes = [], None, []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = f"{r[i]} {units[i]}".strip()
        out.append(d)
        if "gemm" not in d["kernel"]:
            continue
        try:
            t = float(r[hdr.index("dram__bytes_read.sum")].replace(",", "")) * (1e9 if "Gbyte" in units[hdr.index("dram__bytes_read.sum")] else 1)
            wb = float(r[hdr.index("dram__bytes_write.sum")].replace(",", "")) * (1e9 if "Gbyte" in units[hdr.index("dram__bytes_write.sum")] else 1)
            dur = float(r[hdr.index("gpu__time_duration.sum")].replace(",", ""))
            tu = units[hdr.index("gpu__time_duration.sum")]
            dur_ms = dur * {"ms": 1.0, "msecond": 1.0, "us": 1e-3, "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6}.get(tu, 1.0)
            grid = r[hdr.index("launch__grid_size")] if "launch__grid_size" in hdr else ""
            passes.append((dur_ms, t + wb, d["kernel"], grid))
            if best is None or dur > best[0]:
                best = (dur, t + wb, d["kernel"])
        except (ValueError, IndexError):
            pass
    with open(os.path.join(ROOT, "profiles", f"{rnd}_ncu_top_kernels_{wl}.jsonl"), "w") as f:
        for d in out:
            f.write(json.dumps(d) + "\n")
    if best:
        path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        try:
            cur = json.load(open(path))
            if not isinstance(cur, dict) or "kernel" in cur:
                cur = {}
        except Exception:
            cur = {}
        # the passes over A (M-major digit GEMM launches: A X and A^T Q); bench.py's roofline.achieved is an
        # average over the step's passes, so the traffic figure is the mean over the captured pass launches
        pl = [x for x in passes if "ozaki_gemm_kernel<1" in x[2]] or passes
        cur[wl] = {"kernel": best[2], "traffic_bytes": sum(x[1] for x in pl) / len(pl),
                   "per_launch": [{"grid": x[3], "ms": x[0], "dram_bytes": x[1]} for x in pl],
                   "source": f"ncu --set full, profiles/{rnd}_ncu_top_kernels_{wl}.jsonl",
                   "note": "mean of dram__bytes_read.sum + dram__bytes_write.sum over the captured pass launches "
                           "(A X and A^T Q)"}
        json.dump(cur, open(path, "w"), indent=1)
    for d in out:
        print(d)


if __name__ == "__main__":
    rnd, wl = sys.argv[1], sys.argv[2]
    steps_total = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    launches(rnd, wl, steps_total)
    ncu_full(rnd, wl)
