"""Product RCM / permutation (C++ host code) against reference fixtures."""

import hashlib
import json
import os

import numpy as np
import pytest

import oracle
import paper_2307_06305_b200 as dg
from conftest import GOLDEN
from paper_2307_06305_b200.errors import DimensionMismatch, NotSquare


def rcm_cases():
    z = np.load(os.path.join(GOLDEN, "rcm.npz"))
    for k in range(int(z["count"])):
        p = f"r{k}_"
        n = int(z[p + "n"])
        a = dg.CsrMatrix(n, n, z[p + "rowptr"], z[p + "colids"], np.ones(len(z[p + "colids"])))
        yield a, z[p + "perm"], int(z[p + "bw_after"])


def test_rcm_matches_reference_permutations():
    count = 0
    for a, perm, bw in rcm_cases():
        p = dg.rcm(a)
        assert np.array_equal(p.perm, perm)
        assert dg.bandwidth(dg.permute_symmetric(a, p)) == bw
        count += 1
    assert count > 60


def test_rcm_c4_matches_reference_hash():
    from paper_2307_06305_b200.workloads import laplacian_2d, scrambled
    with open(os.path.join(GOLDEN, "c4_rcm.json")) as f:
        g = json.load(f)
    mixed, _ = scrambled(laplacian_2d(g["nx"]), seed=g["scramble_seed"])
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a, np.int64).tobytes()).hexdigest()
    assert sha(mixed.colids) == g["scrambled_colids_sha256"]
    p = dg.rcm(mixed)
    assert sha(p.perm) == g["perm_sha256"]
    assert dg.bandwidth(dg.permute_symmetric(mixed, p)) == g["bandwidth_rcm"]


def test_permute_matches_oracle_and_dense():
    rng = np.random.default_rng(5)
    for _ in range(15):
        n = int(rng.integers(2, 30))
        t = int(rng.integers(0, n * n // 3 + 1))
        a = dg.csr_from_triplets(dg.TripletMatrix(n, n, rng.integers(0, n, t),
                                                  rng.integers(0, n, t), rng.uniform(-1, 1, t)))
        order = rng.permutation(n)
        p = dg.Permutation.from_new_to_old(order)
        b = dg.permute_symmetric(a, p)
        rp, ci, v = oracle.permute(n, a.rowptr, a.colids, a.values, order)
        assert np.array_equal(b.rowptr, rp) and np.array_equal(b.colids, ci)
        assert np.array_equal(b.values, v)
        assert b.rowptr.dtype == a.rowptr.dtype and b.colids.dtype == a.colids.dtype
        d = dg.permute_symmetric(dg.to_dacsr(a, 16), p)
        assert isinstance(d, dg.DacsrMatrix) and dg.to_csr(d, 32) == b


def test_adjacency_and_errors():
    a = dg.csr_from_triplets(dg.TripletMatrix.from_entries(
        4, 4, [(0, 0, 1.0), (1, 2, 2.0), (2, 1, 3.0), (2, 3, 4.0), (3, 3, 5.0)]))
    adj = dg.symmetrized_adjacency(a)
    assert [adj.neighbors(i).tolist() for i in range(4)] == [[], [2], [1, 3], [2]]
    rect = dg.csr_from_triplets(dg.TripletMatrix.from_entries(2, 3, [(0, 2, 1.0)]))
    with pytest.raises(NotSquare):
        dg.symmetrized_adjacency(rect)
    with pytest.raises(DimensionMismatch):
        dg.permute_symmetric(rect, dg.Permutation.identity(2))
    with pytest.raises(DimensionMismatch):
        dg.permute_symmetric(a, dg.Permutation.identity(3))
    with pytest.raises(ValueError):
        dg.Permutation(np.array([0, 0]), np.array([0, 1]))


def test_da_input_is_reordered_by_its_absolute_pattern():
    """The reference's reorder functions read ``a.colids`` as columns
    (reorder.py:78-79, 213-214), which for a DacsrMatrix are offsets: there,
    DA-CSR input is silently treated as a different matrix.  Here the DA
    offsets are turned back into absolute columns first (a deliberate
    difference): RCM of a DA-CSR matrix is the RCM of the
    matrix it stores, and permuting it equals converting the permuted CSR."""
    from paper_2307_06305_b200.workloads import laplacian_2d
    rng = np.random.default_rng(5)
    a = laplacian_2d(12)
    shuffle = dg.Permutation.from_new_to_old(rng.permutation(a.nrows))
    b = dg.permute_symmetric(a, shuffle)          # a wide-band CSR matrix
    d = dg.to_dacsr(b, 16)
    p_csr, p_da = dg.rcm(b), dg.rcm(d)
    assert np.array_equal(p_csr.perm, p_da.perm)
    adj_c, adj_d = dg.symmetrized_adjacency(b), dg.symmetrized_adjacency(d)
    assert np.array_equal(adj_c.indptr, adj_d.indptr) and np.array_equal(adj_c.indices, adj_d.indices)
    out = dg.permute_symmetric(d, p_da)
    assert isinstance(out, dg.DacsrMatrix) and out.iindex_width == 16
    assert dg.to_csr(out, 32) == dg.permute_symmetric(b, p_csr)
