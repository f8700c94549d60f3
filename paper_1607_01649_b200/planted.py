"""planted_matrix — the reference's fixture recipe (proj/src/diagnostics.cpp:124-136)
at BASELINE configuration sizes, row block by row block.

The reference builds A = U diag(sigma) V^T with U, V the Householder Q factors
(householder_qr, dense.cpp:375-400; R's diagonal is non-negative, make_reflector
:328-353) of gaussian(seed, "testmat.u", m, r) and gaussian(seed, "testmat.v",
n, r). Its O(m r^2) single-threaded Householder sweep takes ~75 min at config 3
(SURVEY.md App. B). Here:

* the Gaussians come from the product's host generator (rfgpu_gaussian_range,
  bitwise the reference stream, element-seekable so a rank draws only its rows);
* the Q factor with non-negative R diagonal is unique, so it is formed as
  CholeskyQR2 (Q = X R1^-1 R2^-1, Grams summed over ranks when row-sharded) —
  the same matrix as the reference's Householder Q to rounding (pinned against
  the compiled reference by tests/test_planted.py, ~1e-15);
* the optional noise term eta * N uses N = gaussian(seed, "noise.N", m, n)
  (the tag is a free choice), streamed column block by column
  block without materialising N.

Fixture generation only (not timed; torch is used for the device arithmetic).
Returns A^T for rows [row0, row1) as an (n, rows) tensor, i.e. the row block
of A column-major with lda = rows (the rfgpu_matrix layout).
"""
from __future__ import annotations

import numpy as np


def _gauss_rows(seed: int, tag: str, m: int, cols: int, row0: int, row1: int) -> np.ndarray:
    """Rows [row0, row1) of gaussian(seed, tag, m, cols) as a column-major (rows, cols) array."""
    from . import _check, _dp, lib
    rows = row1 - row0
    out = np.empty((rows, cols), order="F")
    if row0 == 0 and row1 == m:
        _check(lib().rfgpu_gaussian(seed, tag.encode(), m, cols, _dp(out.reshape(-1, order="F"))))
        return out
    flat = out.reshape(-1, order="F")
    for j in range(cols):
        col = flat[j * rows:(j + 1) * rows]
        _check(lib().rfgpu_gaussian_range(seed, tag.encode(), j * m + row0, rows, _dp(col)))
    return out


def _q_factor(torch, x, allreduce=None):
    """Q of the thin QR with non-negative R diagonal (CholeskyQR2; x row-sharded when allreduce is given)."""
    for _ in range(2):
        g = x.T @ x
        if allreduce is not None:
            allreduce(g)
        r = torch.linalg.cholesky(g, upper=True)
        x = torch.linalg.solve_triangular(r, x, upper=True, left=False)
    return x


def planted_matrix(m: int, n: int, sigma, seed: int, noise: float = 0.0, row0: int = 0, row1: int | None = None,
                   device="cpu", allreduce=None, noise_tag: str = "noise.N"):
    """Rows [row0, row1) of planted_matrix(m, n, sigma, seed) + noise * gaussian(seed, noise_tag, m, n),
    returned transposed: an (n, row1 - row0) float64 torch tensor on `device`. allreduce(tensor) sums a
    tensor over ranks in place when the rows are sharded (the Q factor of U needs the summed Gram)."""
    import torch
    row1 = m if row1 is None else row1
    sig = np.asarray(sigma, dtype=np.float64)
    r = len(sig)
    if r > min(m, n):
        raise ValueError("planted_matrix: spectrum longer than min(m,n)")
    dev = torch.device(device)
    u = torch.from_numpy(_gauss_rows(seed, "testmat.u", m, r, row0, row1)).to(dev)
    u = _q_factor(torch, u, allreduce if (row0, row1) != (0, m) else None)
    v = _q_factor(torch, torch.from_numpy(_gauss_rows(seed, "testmat.v", n, r, 0, n)).to(dev))
    at = (v * torch.from_numpy(sig).to(dev)) @ u.T  # n x rows = (U diag(s) V^T)^T for these rows
    del u, v
    if noise:
        rows = row1 - row0
        blk = max(1, min(n, (1 << 27) // max(1, rows)))  # <= 1 GiB of noise per host block
        for j0 in range(0, n, blk):
            j1 = min(n, j0 + blk)
            if row0 == 0 and row1 == m:
                nb = np.empty((rows, j1 - j0), order="F")
                from . import _check, _dp, lib
                _check(lib().rfgpu_gaussian_range(seed, noise_tag.encode(), j0 * m, (j1 - j0) * m,
                                                  _dp(nb.reshape(-1, order="F"))))
            else:
                nb = _gauss_cols(seed, noise_tag, m, row0, row1, j0, j1)
            at[j0:j1].add_(torch.from_numpy(nb.T).to(dev), alpha=noise)
    return at


def _gauss_cols(seed, tag, m, row0, row1, j0, j1):
    from . import _check, _dp, lib
    rows = row1 - row0
    out = np.empty((rows, j1 - j0), order="F")
    flat = out.reshape(-1, order="F")
    for j in range(j0, j1):
        _check(lib().rfgpu_gaussian_range(seed, tag.encode(), j * m + row0, rows,
                                          _dp(flat[(j - j0) * rows:(j - j0 + 1) * rows])))
    return out


def spectrum(kind: str, r: int) -> np.ndarray:
    """The BASELINE.json configs' planted spectra."""
    j = np.arange(1, r + 1, dtype=np.float64)
    if kind == "pow1.5":   # config 3: s_j = j^-1.5
        return j ** -1.5
    if kind == "exp20":    # config 2: s_j = exp(-j/20)
        return np.exp(-j / 20.0)
    if kind == "pow2":     # config 1: s_j = 1/j^2
        return 1.0 / j ** 2
    if kind == "exp100":   # config 4: s_j = exp(-j/100)
        return np.exp(-j / 100.0)
    if kind == "decade6":  # config 5: s_j = 10^(-6 (j-1)/999)
        return 10.0 ** (-6.0 * (j - 1) / (r - 1))
    raise ValueError(kind)
