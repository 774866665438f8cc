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
