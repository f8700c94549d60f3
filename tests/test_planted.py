"""CPU: the config-size fixture generator (paper_1607_01649_b200/planted.py)
reproduces the reference recipe planted_matrix (diagnostics.cpp:124-136) —
the compiled reference's bytes to rounding — whole and row block by row
block (the row-sharded form bench.py and the config tests use)."""
import numpy as np
import pytest
import torch

from paper_1607_01649_b200 import planted as pl


@pytest.mark.parametrize("m,n,r", [(700, 300, 100), (257, 513, 257)])
def test_planted_matches_reference_recipe(ref, m, n, r):
    sig = pl.spectrum("pow1.5", r)
    want = ref.planted(m, n, sig, 1)
    got = pl.planted_matrix(m, n, sig, 1).numpy().T
    assert np.max(np.abs(got - want)) <= 1e-14 * np.max(np.abs(want))


def test_planted_row_blocks_match_whole(ref):
    m, n, r = 901, 200, 60
    sig = pl.spectrum("exp20", r)
    whole = pl.planted_matrix(m, n, sig, 3, noise=1e-6).numpy().T
    bounds = [0, 300, 301, 901]

    u_full = pl._gauss_rows(3, "testmat.u", m, r, 0, m)
    for a, b in zip(bounds[:-1], bounds[1:]):
        part = pl._gauss_rows(3, "testmat.u", m, r, a, b)
        assert np.array_equal(part, u_full[a:b])
    noise = pl._gauss_cols(3, "noise.N", m, 0, m, 0, n)
    noise_blk = pl._gauss_cols(3, "noise.N", m, 300, 901, 5, 17)
    assert np.array_equal(noise_blk, noise[300:901, 5:17])
    want = ref.planted(m, n, sig, 3) + 1e-6 * noise
    assert np.max(np.abs(whole - want)) <= 1e-14 * np.max(np.abs(want))


def test_spectra():
    assert pl.spectrum("decade6", 1000)[-1] == pytest.approx(1e-6)
    assert pl.spectrum("pow2", 3)[2] == pytest.approx(1 / 9)


def _planted_worker(rank, world, port, out):
    import os
    import sys
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1607_01649_b200 import planted as p
    m, n = 777, 160
    r0, r1 = m * rank // world, m * (rank + 1) // world
    at = p.planted_matrix(m, n, p.spectrum("pow1.5", 90), 2, noise=1e-8, row0=r0, row1=r1,
                          allreduce=lambda t: dist.all_reduce(t))
    out.put((rank, r0, r1, at.numpy().copy()))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_planted_row_sharded_world2_matches_whole():
    """bench.py's multi-rank generator: every rank builds only its rows (distributed CholeskyQR2 of the
    reference Gaussian), and together they are the whole planted matrix."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_planted_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    parts = sorted([q.get(timeout=240) for _ in range(2)])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    got = np.hstack([at for _, _, _, at in parts]).T  # (m, n)
    whole = pl.planted_matrix(777, 160, pl.spectrum("pow1.5", 90), 2, noise=1e-8).numpy().T
    assert np.max(np.abs(got - whole)) <= 1e-14 * np.max(np.abs(whole))
