"""GPU parity for the interpolative decompositions (BASELINE config 5 family).

North star: pivot indices must match the reference EXACTLY; interpolation
matrix Z within 1e-8. Reference tests mirrored: proj/tests/test_lowrank.cpp
:187-307 (column / row ID, CUR), proj/tests/test_dense.cpp:118-165 (cpqr).
"""
import os

import numpy as np
import pytest

import paper_1607_01649_b200 as rf

pytestmark = pytest.mark.gpu
FIX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_fixtures.npz")


def c5_spectrum(r):
    return 10.0 ** (-6.0 * np.arange(r) / (r - 1))


def test_col_id_matches_golden_fixture(ctx):
    fx = np.load(FIX)
    f = rf.id_deterministic(fx["cur_Y"], 20, ctx=ctx)
    assert np.array_equal(f.Js, fx["cur_Js"])
    assert np.abs(f.Z - fx["cur_Z"]).max() < 1e-8


def test_row_sketch_matches_oracle(ctx, port):
    a = port.planted(700, 500, c5_spectrum(300), 3)
    y = rf.row_sketch(a, 40, 3, ctx=ctx)
    want = port.multiply(port.gaussian(3, "cur.G", 40, 700), a)
    assert np.abs(y - want).max() <= 1e-13 * np.abs(want).max()


@pytest.mark.parametrize("m,n,k,p", [(2048, 2048, 100, 20), (1500, 3000, 200, 20), (4096, 4096, 300, 20)])
def test_cur_column_id_pivots_exact(ctx, port, m, n, k, p):
    a = port.planted(m, n, c5_spectrum(min(1000, m, n)), 1)
    js_w, z_w, tr_w, y = port.cur_col_id(a, k, p, 1)
    f = rf.id_deterministic(y, k, ctx=ctx)
    assert not f.rank_truncated and not tr_w
    assert np.array_equal(f.Js, js_w)
    assert np.abs(f.Z - z_w).max() < 1e-8
    # Z(:, Js) = I exactly (test_lowrank.cpp:194-199)
    assert np.array_equal(f.Z[:, f.Js], np.eye(k))


def test_randomized_cur_matches_oracle(ctx, port):
    a = port.planted(1200, 1000, c5_spectrum(500), 2)
    want = port.randomized_cur(a, 60, 20, 0, 2)
    got = rf.randomized_cur(a, 60, 20, 0, 2, ctx=ctx)
    assert np.array_equal(got.Js, want.Js)
    assert np.array_equal(got.Is, want.Is)
    assert np.abs(got.U - want.U).max() <= 1e-8 * np.abs(want.U).max()
    assert abs(got.cond_C - want.cond_C) <= 1e-8 * want.cond_C
    assert abs(got.cond_R - want.cond_R) <= 1e-8 * want.cond_R
    assert got.warning == want.warning


def test_randomized_cur_exact_rank_reconstruction(ctx, port):
    # test_lowrank.cpp:276-307
    a = port.planted(25, 18, 0.6 ** np.arange(5.0), 33)
    f = rf.randomized_cur(a, 5, 5, 1, 3, ctx=ctx)
    assert len(f.Js) == 5 and len(f.Is) == 5 and f.U.shape == (5, 5)
    rec = a[:, f.Js] @ f.U @ a[f.Is, :]
    assert np.linalg.norm(a - rec) < 1e-8 * np.linalg.norm(a)
    assert len(set(f.Js.tolist())) == 5 and f.cond_C > 0 and f.cond_R > 0 and not f.warning


def test_randomized_id_matches_oracle(ctx, port):
    a = port.planted(800, 600, c5_spectrum(400), 4)
    for q in (0, 1):
        is_w, x_w, _ = port.randomized_id(a, 50, 10, q, 5)
        f = rf.randomized_id(a, 50, 10, q, 5, ctx=ctx)
        assert np.array_equal(f.Is, is_w)
        assert np.abs(f.X - x_w).max() < 1e-8


def test_id_reports_truncation(ctx, port):
    # test_lowrank.cpp:240-247: numerical rank 4 < k = 8
    a = port.planted(16, 12, 0.5 ** np.arange(4.0), 2)
    js_w, z_w, tr_w = port.id_col(a, 8)
    f = rf.id_deterministic(a, 8, ctx=ctx)
    assert f.rank_truncated and tr_w
    assert np.array_equal(f.Js, js_w)
    assert np.abs(f.Z - z_w).max() < 1e-8


def test_cpqr_known_answer_diag(ctx):
    # test_dense.cpp:118-132: diag(1,2,3) pivots [2,1,0]
    f = rf.id_deterministic(np.diag([1.0, 2.0, 3.0]), 3, ctx=ctx)
    assert list(f.Js) == [2, 1, 0]


def test_id_validation(ctx):
    with pytest.raises(rf.ParameterError):
        rf.id_deterministic(np.ones((5, 4)), 0, ctx=ctx)
    with pytest.raises(rf.ParameterError):
        rf.id_deterministic(np.ones((5, 4)), 5, ctx=ctx)
