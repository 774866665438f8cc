"""Bandwidth reduction: reverse Cuthill–McKee and symmetric permutation.

Same API and results as the reference (/root/reference/pkg/src/dacsr/
reorder.py): ``Permutation`` (17-55), ``Adjacency`` (58-67),
``symmetrized_adjacency`` (70-97), ``rcm`` (146-197, bit-identical
permutations — every tie broken by ascending degree then ascending index)
and ``permute_symmetric`` (200-220).  The graph work runs in the native
library's C++ host code (csrc/host_reorder.cpp) instead of a pure-Python
BFS: config C4 (n = 4.19M) takes seconds instead of ~92 s.
"""

from dataclasses import dataclass

import numpy as np

from . import _native
from .core import CsrMatrix, DacsrMatrix, _trusted, index_dtype
from .errors import DimensionMismatch, NotSquare


@dataclass(frozen=True, eq=False)
class Permutation:
    """Bijection on [0, n): ``perm[new] = old`` and ``inv[old] = new``."""

    perm: np.ndarray
    inv: np.ndarray

    def __post_init__(self):
        p = np.asarray(self.perm, dtype=np.int64)
        q = np.asarray(self.inv, dtype=np.int64)
        n = len(p)
        if len(q) != n:
            raise ValueError("perm and inv must have equal length")
        ident = np.arange(n, dtype=np.int64)
        if not np.array_equal(np.sort(p), ident):
            raise ValueError("perm is not a bijection on [0, n)")
        if not np.array_equal(q[p], ident):
            raise ValueError("inv does not invert perm")
        for arr in (p, q):
            if arr.flags.writeable:
                arr.flags.writeable = False
        object.__setattr__(self, "perm", p)
        object.__setattr__(self, "inv", q)

    @classmethod
    def from_new_to_old(cls, order):
        p = np.asarray(order, dtype=np.int64)
        q = np.empty(len(p), dtype=np.int64)
        q[p] = np.arange(len(p), dtype=np.int64)
        return cls(p, q)

    @classmethod
    def identity(cls, n):
        return cls(np.arange(n, dtype=np.int64), np.arange(n, dtype=np.int64))

    @property
    def n(self):
        return len(self.perm)


@dataclass(frozen=True, eq=False)
class Adjacency:
    """Undirected graph in CSR layout; sorted neighbour lists, no self-loops."""

    n: int
    indptr: np.ndarray
    indices: np.ndarray

    def neighbors(self, u):
        return self.indices[self.indptr[u]:self.indptr[u + 1]]


def _ptr(a):
    return a.ctypes.data_as(_native.ctypes.c_void_p)


def _absolute_columns(a):
    cols = a.colids.astype(np.int64)
    if isinstance(a, DacsrMatrix):
        from .core import entry_rows
        cols += entry_rows(a.rowptr)
    return np.ascontiguousarray(cols)


def symmetrized_adjacency(a):
    """Graph of the pattern of A + A^T with self-loops removed."""
    if a.nrows != a.ncols:
        raise NotSquare(f"adjacency requires a square matrix, got {a.nrows}x{a.ncols}")
    n = a.nrows
    rp = np.ascontiguousarray(a.rowptr, dtype=np.int64)
    cols = _absolute_columns(a)
    indptr = np.zeros(n + 1, dtype=np.int64)
    L = _native.lib()
    _native.check(L.dacsr_host_adjacency(n, _ptr(rp), _ptr(cols), _ptr(indptr), None),
                  "dacsr_host_adjacency")
    indices = np.empty(int(indptr[-1]), dtype=np.int64)
    _native.check(L.dacsr_host_adjacency(n, _ptr(rp), _ptr(cols), _ptr(indptr), _ptr(indices)),
                  "dacsr_host_adjacency")
    indptr.flags.writeable = False
    indices.flags.writeable = False
    return Adjacency(n, indptr, indices)


def rcm(a):
    """Reverse Cuthill–McKee permutation of a square matrix (new → old)."""
    adj = symmetrized_adjacency(a)
    perm = np.empty(adj.n, dtype=np.int64)
    _native.check(_native.lib().dacsr_host_rcm(adj.n, _ptr(adj.indptr), _ptr(adj.indices),
                                               _ptr(perm)), "dacsr_host_rcm")
    return Permutation.from_new_to_old(perm)


def permute_symmetric(a, p):
    """result(r, c) = a(perm[r], perm[c]); nnz, widths and canonical form kept."""
    if a.nrows != a.ncols:
        raise DimensionMismatch(
            f"symmetric permutation requires a square matrix, got {a.nrows}x{a.ncols}")
    if p.n != a.nrows:
        raise DimensionMismatch(f"permutation of size {p.n} does not match dimension {a.nrows}")
    n = a.nrows
    src = a if isinstance(a, CsrMatrix) else None
    if src is None:  # DA-CSR input: permute its absolute pattern, keep widths
        cols = _absolute_columns(a)
    else:
        cols = np.ascontiguousarray(a.colids, dtype=np.int64)
    rp = np.ascontiguousarray(a.rowptr, dtype=np.int64)
    vals = np.ascontiguousarray(a.values)
    out_rp = np.empty(n + 1, dtype=np.int64)
    out_cols = np.empty(a.nnz, dtype=np.int64)
    out_vals = np.empty(a.nnz, dtype=vals.dtype)
    perm = np.ascontiguousarray(p.perm, dtype=np.int64)
    _native.check(_native.lib().dacsr_host_permute(
        n, _ptr(rp), _ptr(cols), _ptr(vals), vals.dtype.itemsize, _ptr(perm), _ptr(out_rp),
        _ptr(out_cols), _ptr(out_vals)), "dacsr_host_permute")
    csr = _trusted(CsrMatrix, n, n, out_rp.astype(a.rowptr.dtype),
                   out_cols.astype(index_dtype(a.iindex_width)) if src is not None
                   else out_cols.astype(np.int64), out_vals)
    if src is not None:
        return csr
    from .core import to_dacsr
    return to_dacsr(csr, a.iindex_width)


__all__ = ["Adjacency", "Permutation", "permute_symmetric", "rcm", "symmetrized_adjacency"]
