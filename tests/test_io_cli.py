"""Matrix files and the CLI front end.

CPU: randfact::read_matrix / write_matrix of the drop-in (host/matrix_io.cpp),
called from a program compiled against the REFERENCE header matrix_io.hpp
(tests/dropin/dropin_probe.cpp, modes io / iow), against the compiled
reference reader / writer (matrix_io.cpp) on the same files: same status class,
same message (path:line), bitwise the same matrix, byte-identical written
files. The CLI (randfact_b200, host/cli.cpp) rejects bad command lines and
files with the reference's exit codes (cli.cpp:459-471) before touching a GPU.

GPU: `factorize` / `bench` reports in the randfact/1 schema (cli.cpp:268-343)
for rsvd / spsvd / id / cur: results against the oracle, errors recomputed on
the device against numpy.
"""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROBE = os.path.join(ROOT, "oracle", "_ref", "dropin_probe")
CLI = os.path.join(ROOT, "paper_1607_01649_b200", "randfact_b200")
needs_probe = pytest.mark.skipif(not os.path.exists(PROBE), reason="dropin_probe not built (needs /root/reference)")

VALID = {
    "array_general.mtx": "%%MatrixMarket matrix array real general\n% comment\n\n3 2\n1.5\n-2\n3e-3\n4\n5.25\n+6\n",
    "array_symmetric.mm": "%%MatrixMarket matrix array real symmetric\n3 3\n1\n2\n3\n4\n5\n6\n",
    "coord_dups.mtx": "%%MatrixMarket matrix coordinate real general\n%x\n3 4 4\n1 1 1.0\n3 4 -2.5\n1 1 0.25\n2 3 7\n",
    "coord_pattern_sym.mtx": "%%MatrixMarket matrix coordinate pattern symmetric\n4 4 3\n1 1\n3 1\n4 2\n",
    "coord_integer.mtx": "%%matrixmarket MATRIX Coordinate INTEGER General\n2 2 2\n1 2 3\n2 1 -4\n",
    "tokens_across_lines.mtx": "%%MatrixMarket matrix array real general\n2\n2 1 2\n3 4\n",
    "plain.csv": "1, 2 ,3\n\n4,5.5,-6e2\r\n",
}
INVALID = {
    "no_banner.mtx": "%MatrixMarket matrix array real general\n1 1\n1\n",
    "complex.mtx": "%%MatrixMarket matrix array complex general\n1 1\n1 0\n",
    "hermitian.mtx": "%%MatrixMarket matrix array real hermitian\n1 1\n1\n",
    "array_pattern.mtx": "%%MatrixMarket matrix array pattern general\n1 1\n",
    "bad_entry.mtx": "%%MatrixMarket matrix array real general\n2 1\n1\nx2\n",
    "nonfinite.mtx": "%%MatrixMarket matrix array real general\n1 1\ninf\n",
    "out_of_range.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n",
    "trailing.mtx": "%%MatrixMarket matrix array real general\n1 1\n1\n2\n",
    "short.mtx": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n",
    "zero_dim.mtx": "%%MatrixMarket matrix array real general\n0 2\n",
    "sym_rect.mtx": "%%MatrixMarket matrix array real symmetric\n2 3\n1\n2\n3\n",
    "neg_index.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 -1\n",
    "empty.mtx": "",
    "ragged.csv": "1,2\n3\n",
    "empty_cell.csv": "1,,2\n",
    "bad_cell.csv": "1,2x\n",
    "empty.csv": "\n\n",
    "unknown.txt": "1\n",
}


def write_files(tmp_path, table):
    out = {}
    for name, text in table.items():
        p = tmp_path / name
        p.write_text(text)
        out[name] = str(p)
    return out


def probe_read(path, tmp_path):
    out = str(tmp_path / "probe_out.bin")
    r = subprocess.run([PROBE, "io", path, out], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr
    line = r.stdout.strip()
    kind, _, rest = line.partition(" ")
    if kind == "OK":
        m, n = map(int, rest.split())
        return 0, "", np.fromfile(out).reshape((m, n), order="F")
    return {"PARSE_ERROR": 2, "PARAM_ERROR": 3}.get(kind, 1), rest, None


@needs_probe
@pytest.mark.parametrize("name", sorted(VALID) + sorted(INVALID))
def test_read_matrix_matches_reference(ref, tmp_path, name):
    path = write_files(tmp_path, {name: {**VALID, **INVALID}[name]})[name]
    st_r, msg_r, a_r = ref.read_matrix(path)
    st_g, msg_g, a_g = probe_read(path, tmp_path)
    assert (st_g, msg_g) == (st_r, msg_r)
    if st_r == 0:
        assert a_g.shape == a_r.shape and np.array_equal(a_g, a_r)
    else:
        assert name in INVALID


@needs_probe
def test_read_matrix_missing_file(ref, tmp_path):
    path = str(tmp_path / "nope.mtx")
    assert probe_read(path, tmp_path)[:2] == ref.read_matrix(path)[:2]


@needs_probe
@pytest.mark.parametrize("ext", [".mtx", ".csv"])
def test_write_matrix_byte_identical(ref, tmp_path, ext):
    a = np.asfortranarray(np.random.default_rng(1).standard_normal((7, 5)) * 10.0 ** np.arange(5))
    a[2, 3] = 0.1
    a[0, 0] = -0.0
    src = str(tmp_path / "a.bin")
    a.reshape(-1, order="F").tofile(src)
    ours, theirs = str(tmp_path / ("ours" + ext)), str(tmp_path / ("ref" + ext))
    r = subprocess.run([PROBE, "iow", src, "7", "5", ours], capture_output=True, text=True, timeout=60)
    assert r.stdout.strip() == "OK", r.stdout + r.stderr
    assert ref.write_matrix(theirs, a)[0] == 0
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    bad = a.copy()
    bad[1, 1] = np.nan
    bad.reshape(-1, order="F").tofile(src)
    r = subprocess.run([PROBE, "iow", src, "7", "5", ours], capture_output=True, text=True, timeout=60)
    st, msg = ref.write_matrix(ours, bad)  # same target path: the message names it
    assert st == 4 and r.stdout.strip() == f"NUMERICAL_ERROR {msg}"


def cli(*args):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=900)


@pytest.mark.parametrize("args,code", [
    ([], 3),
    (["frobnicate"], 3),
    (["factorize", "--algo", "rsvd"], 3),
    (["factorize", "--algo", "nosuch", "--in", "x.mtx"], 3),
    (["factorize", "--algo", "rsvd", "--in", "x.mtx", "--k", "0"], 3),
    (["factorize", "--algo", "rsvd", "--in", "x.mtx", "--bogus", "1"], 3),
    (["bench", "--in", "x.mtx"], 3),
])
def test_cli_rejects_bad_command_lines(args, code):
    r = cli(*args)
    assert r.returncode == code, r.stdout + r.stderr
    assert "error:" in r.stderr


def test_cli_file_errors_before_any_device_work(tmp_path):
    files = write_files(tmp_path, {"bad.mtx": INVALID["bad_entry.mtx"], "a.txt": "1\n",
                                   "ok.mtx": VALID["array_general.mtx"]})
    r = cli("factorize", "--algo", "rsvd", "--in", files["bad.mtx"], "--k", "1", "--p", "0")
    assert r.returncode == 2 and f"{files['bad.mtx']}:4: bad matrix entry 'x2'" in r.stderr
    r = cli("factorize", "--algo", "rsvd", "--in", files["a.txt"])
    assert r.returncode == 3 and "unknown matrix file extension" in r.stderr
    r = cli("factorize", "--algo", "rsvd", "--in", str(tmp_path / "missing.mtx"))
    assert r.returncode == 2 and "cannot open" in r.stderr
    r = cli("factorize", "--algo", "hqrrp", "--in", files["ok.mtx"])  # a reference algorithm off the B200 path
    assert r.returncode == 3 and "outside the B200 hot path" in r.stderr


# ------------------------------------------------------------------------------------ GPU ---
def write_mtx(path, a):
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix array real general\n")
        f.write(f"{a.shape[0]} {a.shape[1]}\n")
        for v in np.asfortranarray(a).reshape(-1, order="F"):
            f.write(f"{v:.17g}\n")


def schema_ok(rep, mode):
    assert rep["schema"] == "randfact/1" and rep["mode"] == mode
    for key in ("input", "params"):
        assert key in rep
    assert set(rep["params"]) >= {"k", "p", "q", "b", "r", "eps", "seed", "keep_oversamples", "reorthonormalize",
                                  "deterministic"}


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["rsvd", "spsvd", "id", "cur"])
def test_cli_factorize_report(port, tmp_path, algo):
    m, n = 300, 240
    sig = 10.0 ** (-4.0 * np.arange(240) / 239.0)
    a = port.planted(m, n, sig, 4) + 1e-9 * port.gaussian(4, "noise.N", m, n)
    path = str(tmp_path / "a.mtx")
    write_mtx(path, a)
    rep_path = str(tmp_path / "rep.json")
    q = ["--q", 0] if algo == "cur" else ["--q", 1, "--reorth"]  # the port restates randomized_cur for q = 0
    r = cli("factorize", "--algo", algo, "--in", path, "--k", 20, "--p", 10, *q, "--seed", 3, "--report", rep_path)
    assert r.returncode == 0, r.stdout + r.stderr
    rep = json.load(open(rep_path))
    schema_ok(rep, "factorize")
    assert rep["algo"] == algo and rep["input"]["rows"] == m and rep["input"]["cols"] == n
    assert rep["input"]["frob"] == pytest.approx(np.linalg.norm(a), rel=1e-12)
    res = rep["results"]
    if algo == "rsvd":
        want = port.rsvd(a, 20, 10, 1, 3, False, True)
        assert res["rank"] == 20
        assert np.max(np.abs(np.array(res["singvals_head"]) - want.D[:10]) / want.D[:10]) <= 1e-10
        approx = (want.U * want.D) @ want.V.T
    elif algo == "spsvd":
        assert res["p_used"] == 10 and res["rank"] == 20
        want = port.single_pass_svd(a, 20, 10, 3, block=32)
        assert np.max(np.abs(np.array(res["singvals_head"]) - want.D[:10]) / want.D[:10]) <= 1e-8
        approx = (want.U * want.D) @ want.V.T
    elif algo == "id":
        is_, x, _ = port.randomized_id(a, 20, 10, 1, 3)
        assert res["rows_head"] == list(is_[:10])
        approx = x @ a[is_, :]
    else:
        want = port.randomized_cur(a, 20, 10, 0, 3)
        assert res["cols_head"] == list(want.Js[:10]) and res["rows_head"] == list(want.Is[:10])
        assert res["cond_C"] == pytest.approx(want.cond_C, rel=1e-8)
        approx = a[:, want.Js] @ want.U @ a[want.Is, :]
    fa = np.linalg.norm(a - approx)
    err = rep["errors"]
    assert err["frob_abs"] == pytest.approx(fa, rel=1e-6, abs=1e-12 * np.linalg.norm(a))
    assert err["frob_rel"] == pytest.approx(err["frob_abs"] / np.linalg.norm(a), rel=1e-12)
    assert err["spectral_probe_abs"] > 0 and "probabilistic upper bound" in err["spectral_probe_note"]
    orc = rep["oracle"]  # max(m, n) <= 320
    sv = np.linalg.svd(a, compute_uv=False)
    assert np.allclose(orc["sigma_head"], sv[:10], rtol=1e-10)
    assert orc["rank_compared"] == res["rank"]
    assert orc["eckart_young_tail_at_rank"] == pytest.approx(np.sqrt(np.sum(sv[res["rank"]:] ** 2)), rel=1e-8)
    assert rep["warnings"] == [] or isinstance(rep["warnings"], list)


@pytest.mark.gpu
def test_cli_bench_report(port, tmp_path):
    a = port.planted(400, 350, 1.0 / np.arange(1, 351) ** 2, 2)
    path = str(tmp_path / "a.csv")
    np.savetxt(path, a, delimiter=",", fmt="%.17g")
    r = cli("bench", "--algos", "rsvd,cur,hqrrp", "--in", path, "--runs", 3, "--k", 10, "--p", 5, "--reorth")
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    schema_ok(rep, "bench")
    assert rep["runs_per_algo"] == 3 and len(rep["runs"]) == 9
    assert [row["seed"] for row in rep["runs"][:3]] == [0, 1, 2]
    assert rep["summary"]["rsvd"]["completed"] == 3 and rep["summary"]["cur"]["completed"] == 3
    assert rep["summary"]["hqrrp"]["completed"] == 0 and "outside the B200 hot path" in rep["runs"][6]["error"]
    want = port.rsvd(a, 10, 5, 0, 0, False, True)
    fr = np.linalg.norm(a - (want.U * want.D) @ want.V.T) / np.linalg.norm(a)
    assert rep["runs"][0]["frob_rel"] == pytest.approx(fr, rel=1e-6)
