"""Seeded synthetic matrices for the BASELINE.json configurations.

The paper measures SuiteSparse matrices, which are not
available here; these generators stand in with the shapes, bandwidths and
value distributions BASELINE.json names:

* C1  ``laplacian_2d(1024)``           5-point, natural order, w = 1024
* C2  ``laplacian_3d(128)``            7-point, w = 16384 (f64 and f32)
* C3  ``banded_poisson(2**24, 32767, 16, 64)``   (device generator)
* C4  ``skewed_rcm_laplacian(2048)``   scrambled → RCM → Pareto skew rows
* C5  ``banded_poisson(2**28, 32767, 8, 32)``    (device generator)

Structured generators emit canonical CSR directly (sorted distinct columns
per row), never via triplets.  ``scrambled`` follows the reference idiom
``Permutation.from_new_to_old(default_rng(seed).permutation(n))``
(/root/reference/pkg/src/dacsr/generate.py:93-97).
"""

import numpy as np

from .core import CsrMatrix, _trusted


def _stencil_csr(shape, stencil, diag_value, off_value, dtype=np.float64):
    """Canonical CSR of a constant-coefficient stencil on a box grid.

    ``shape`` is the grid extent (slowest axis first, natural row order);
    ``stencil`` lists (axis, step) pairs.  Column order within a row is the
    ascending linear offset, which is the order of ``stencil`` sorted by
    offset.
    """
    shape = tuple(int(s) for s in shape)
    n = int(np.prod(shape))
    strides = [int(np.prod(shape[a + 1:])) for a in range(len(shape))]
    coords = np.indices(shape, dtype=np.int64).reshape(len(shape), n)
    taps = sorted(((step * strides[axis], axis, step) for axis, step in stencil),
                  key=lambda t: t[0])
    valid = []
    for off, axis, step in taps:
        if step == 0:
            valid.append(np.ones(n, dtype=bool))
        else:
            c = coords[axis] + step
            valid.append((c >= 0) & (c < shape[axis]))
    valid = np.stack(valid)                       # [taps, n]
    counts = valid.sum(axis=0)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    nnz = int(rowptr[-1])
    slot = np.cumsum(valid, axis=0) - 1           # position inside the row
    colids = np.empty(nnz, dtype=np.int64)
    values = np.empty(nnz, dtype=dtype)
    rows = np.arange(n, dtype=np.int64)
    for t, (off, axis, step) in enumerate(taps):
        m = valid[t]
        dst = rowptr[:-1][m] + slot[t][m]
        colids[dst] = rows[m] + off
        values[dst] = diag_value if step == 0 else off_value
    return _trusted(CsrMatrix, n, n, rowptr.astype(np.int32),
                    colids.astype(np.int32), values)


def laplacian_2d(nx, dtype=np.float64):
    """5-point Laplacian on an nx×nx grid: 4 on the diagonal, −1 beside it."""
    st = [(0, -1), (1, -1), (0, 0), (1, 1), (0, 1)]
    return _stencil_csr((nx, nx), st, 4.0, -1.0, dtype)


def laplacian_3d(nx, dtype=np.float64):
    """7-point Laplacian on an nx³ grid: 6 on the diagonal, −1 beside it."""
    st = [(0, -1), (1, -1), (2, -1), (0, 0), (2, 1), (1, 1), (0, 1)]
    return _stencil_csr((nx, nx, nx), st, 6.0, -1.0, dtype)


def laplacian_3d_box(shape, dtype=np.float64):
    """7-point Laplacian on a box grid ``shape`` = (nz, ny, nx), slowest axis
    first: the largest offset is ny*nx, so a long thin box (1024, 128, 128)
    gives C2's stencil and int16 offsets at 8 times C2's size — out of L2."""
    st = [(0, -1), (1, -1), (2, -1), (0, 0), (2, 1), (1, 1), (0, 1)]
    return _stencil_csr(tuple(shape), st, 6.0, -1.0, dtype)


def uniform_x(n, seed, low=-1.0, high=1.0):
    """x ~ U[low, high) float64 from ``default_rng(seed)``."""
    return np.random.default_rng(seed).uniform(low, high, n)


def normal_x(n, seed):
    """x ~ N(0, 1) float64 from ``default_rng(seed)``."""
    return np.random.default_rng(seed).standard_normal(n)


def scrambled(a, seed=0):
    """Random symmetric permutation of ``a``; returns (matrix, permutation)."""
    from .reorder import Permutation, permute_symmetric
    p = Permutation.from_new_to_old(
        np.random.default_rng(seed).permutation(a.nrows).astype(np.int64))
    return permute_symmetric(a, p), p


__all__ = ["laplacian_2d", "laplacian_3d", "normal_x", "scrambled", "uniform_x"]


def add_skew_rows(a, frac=0.01, alpha=1.5, x_m=1.0, cap=4096, band=None, seed=0):
    """Give ``frac`` of the rows power-law extra entries (config C4).

    Selected rows (``default_rng(seed).choice(n, round(frac*n))``) receive
    ``min(cap, floor(x_m * Pareto(alpha)))`` extra distinct columns inside
    ``[r - band, r + band] ∩ [0, ncols)`` (band defaults to the matrix's
    bandwidth, so the int16 fit is preserved) with N(0, 1) values.
    Pareto(alpha) with scale x_m is ``x_m * (1 + rng.pareto(alpha))``.
    """
    from .core import bandwidth, entry_rows
    rng = np.random.default_rng(seed)
    n, m = a.nrows, a.ncols
    band = bandwidth(a) if band is None else int(band)
    rows = np.sort(rng.choice(n, size=int(round(frac * n)), replace=False))
    extra = np.minimum(cap, np.floor(x_m * (1.0 + rng.pareto(alpha, len(rows))))).astype(np.int64)
    add_r, add_c = [], []
    rp = a.rowptr.astype(np.int64)
    for r, k in zip(rows.tolist(), extra.tolist()):
        lo, hi = max(0, r - band), min(m - 1, r + band)
        have = a.colids[rp[r]:rp[r + 1]].astype(np.int64)
        window = np.setdiff1d(np.arange(lo, hi + 1, dtype=np.int64), have, assume_unique=True)
        k = min(k, len(window))
        add_r.append(np.full(k, r, dtype=np.int64))
        add_c.append(np.sort(rng.choice(window, size=k, replace=False)))
    add_r = np.concatenate(add_r) if add_r else np.zeros(0, np.int64)
    add_c = np.concatenate(add_c) if add_c else np.zeros(0, np.int64)
    add_v = rng.standard_normal(len(add_r)).astype(a.values.dtype)
    r_all = np.concatenate([entry_rows(a.rowptr), add_r])
    c_all = np.concatenate([a.colids.astype(np.int64), add_c])
    v_all = np.concatenate([a.values, add_v])
    order = np.lexsort((c_all, r_all))
    counts = np.bincount(r_all, minlength=n)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    return _trusted(CsrMatrix, n, m, rowptr.astype(a.rowptr.dtype),
                    c_all[order].astype(a.colids.dtype), v_all[order])


def skewed_rcm_laplacian(nx=2048, scramble_seed=4, skew_seed=5, frac=0.01, alpha=1.5,
                         x_m=1.0, cap=4096):
    """Config C4: scrambled nx² Laplacian → RCM → Pareto skew rows in band.

    Returns (matrix, info) where info records the seeds, bandwidths and the
    RCM permutation (new → old) for parity checks.
    """
    from .core import bandwidth
    from .reorder import permute_symmetric, rcm
    lap = laplacian_2d(nx)
    mixed, _ = scrambled(lap, seed=scramble_seed)
    perm = rcm(mixed)
    ordered = permute_symmetric(mixed, perm)
    w = bandwidth(ordered)
    out = add_skew_rows(ordered, frac=frac, alpha=alpha, x_m=x_m, cap=cap, band=w, seed=skew_seed)
    info = {"nx": nx, "scramble_seed": scramble_seed, "skew_seed": skew_seed, "frac": frac,
            "alpha": alpha, "x_m": x_m, "cap": cap, "bandwidth_scrambled": bandwidth(mixed),
            "bandwidth_rcm": w, "perm": perm.perm}
    return out, info


def poisson_cdf(lam, kmax):
    """P(K <= k) for k = 0..kmax-1 of Poisson(lam), float64 (host-computed
    table shared by the device generator and its CPU checker)."""
    import math
    out = np.empty(kmax, dtype=np.float64)
    acc = 0.0
    for k in range(kmax):
        acc += math.exp(k * math.log(lam) - lam - math.lgamma(k + 1))
        out[k] = acc
    return out


def normal_table(points=4096):
    """``points + 1`` quantiles of N(0, 1) at (i + 0.5) / (points + 1)."""
    from statistics import NormalDist
    nd = NormalDist()
    return np.array([nd.inv_cdf((i + 0.5) / (points + 1)) for i in range(points + 1)],
                    dtype=np.float64)


BANDED_CONFIGS = {
    # name: (n, half bandwidth, lambda, kmax, seed)
    "c3": (1 << 24, 32767, 16.0, 64, 2023),
    "c5": (1 << 28, 32767, 8.0, 32, 2028),
}
