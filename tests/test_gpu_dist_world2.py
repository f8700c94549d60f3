"""GPU, world size 2 on ONE B200: librfgpu's own row-sharded multi-GPU code.

Two processes, each a rank holding a contiguous row block of A (the sharding
of SURVEY.md §8(e) and bench.py), call the library through the C ABI; the
sums over ranks (the n x l pass products A^T Y / B^T, the l x l Grams of the
distributed CholeskyQR2, ||A||_F^2, global_rows, the zero-padded gathers of
the ID / CUR, Yr and the core products of the single pass) run through the
host-staged reduction backend (rfgpu_ctx_create_hostsum) with a gloo
all_reduce, because NCCL cannot place two ranks on one device. Everything
else is the code the NCCL context runs. Each rank's result is compared with
the single-process call on the whole A (tests/dist_worker.py):

* rsvd / power_range, both orth modes, FP64 DMMA and INT8-digit passes:
  singular values 1e-10 relative, U rows and V 1e-8 (sign-aligned), same
  kept rank (reference rangefinder.cpp:63-80, lowrank.cpp:74-96);
* exact-rank input (distributed Gram-Schmidt drop rule, dense.cpp:402-431);
* randomized_id / randomized_cur: pivots identical, X rows / U 1e-8
  (lowrank.cpp:312-372);
* streamed single_pass_svd: 1e-10 / 1e-8 (lowrank.cpp:160-220).

The numpy gloo mirrors (test_dist_gloo*.py) stay as CPU design pins.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "dist_worker.py")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_world2(case, tmp_path):
    port = str(free_port())
    outs = [str(tmp_path / f"{case}_{r}.json") for r in range(2)]
    procs = [subprocess.Popen([sys.executable, WORKER, str(r), "2", port, outs[r], case], stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True, cwd=ROOT) for r in range(2)]
    logs = []
    for p in procs:
        try:
            logs.append(p.communicate(timeout=600)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
    for r, p in enumerate(procs):
        assert p.returncode == 0, f"rank {r} failed:\n{logs[r][-4000:]}"
    return [json.load(open(o)) for o in outs]


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["rsvd_reorth_dmma", "rsvd_reorth_digits", "rsvd_plain_dmma", "rsvd_plain_digits"])
def test_world2_rsvd_matches_single_process(case, tmp_path):
    for r in run_world2(case, tmp_path):
        assert r["host_sums"] > 0  # the distributed branches ran
        assert r["rank_got"] == r["rank_want"]
        tol = 1e-10 if "reorth" in case else 1e-6  # plain mode: the sketch's intrinsic noise floor
        assert r["sigma"] <= tol, r
        if "reorth" in case:
            assert r["V"] <= 1e-8 and r["U_rows"] <= 1e-8, r
        assert r["range_cols"][0] == r["range_cols"][1]
        assert r["resid_rel"] <= 1e-6 and r["B"] <= 1e-8, r


@pytest.mark.gpu
def test_world2_exact_rank_drops_columns(tmp_path):
    for r in run_world2("exact_rank", tmp_path):
        assert r["rank_got"] == r["rank_want"] == 10, r
        assert r["sigma"] <= 1e-9 and r["U_rows"] <= 1e-8, r


@pytest.mark.gpu
def test_world2_randomized_id(tmp_path):
    for r in run_world2("id", tmp_path):
        assert r["pivots_equal"], r
        assert r["X_rows"] <= 1e-8, r


@pytest.mark.gpu
def test_world2_randomized_cur(tmp_path):
    for r in run_world2("cur", tmp_path):
        assert r["js_equal"] and r["is_equal"], r
        assert r["U"] <= 1e-8 and max(r["cond"]) <= 1e-8, r


@pytest.mark.gpu
def test_world2_single_pass_stream(tmp_path):
    for r in run_world2("single_pass", tmp_path):
        assert r["sigma"] <= 1e-10, r
        assert r["V"] <= 1e-8 and r["U_rows"] <= 1e-8, r
