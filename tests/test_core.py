"""Formats and conversions against reference-generated fixtures."""

import os

import numpy as np
import pytest

import paper_2307_06305_b200 as dg
from conftest import GOLDEN
from paper_2307_06305_b200.errors import (BandwidthExceedsIndexRange, EntryOutOfBounds,
                                          IndexRangeExceeded)


def test_conversions_golden():
    z = np.load(os.path.join(GOLDEN, "conversions.npz"))
    for k in range(int(z["count"])):
        p = f"c{k}_"
        nr, nc, iw = (int(v) for v in z[p + "shape"])
        a = dg.CsrMatrix(nr, nc, z[p + "rowptr"], z[p + "colids"], z[p + "values"])
        assert dg.bandwidth(a) == int(z[p + "bandwidth"])
        if int(z[p + "ok"]):
            d = dg.to_dacsr(a, iw)
            assert d.colids.dtype == z[p + "offsets"].dtype
            assert np.array_equal(d.colids, z[p + "offsets"])
            assert dg.bandwidth(d) == int(z[p + "bandwidth"])
            assert dg.to_csr(d, 32) == a
        else:
            with pytest.raises(BandwidthExceedsIndexRange):
                dg.to_dacsr(a, iw)


def test_corpus_construction_matches_reference():
    """csr_from_triplets on the golden inputs reproduces the reference's
    canonical arrays (duplicates summed, explicit zeros kept)."""
    from test_oracle import CORPUS
    for c in CORPUS[:60]:
        a = dg.CsrMatrix(c["nrows"], c["ncols"], c["rowptr"], c["colids"], c["values"])
        rows = np.repeat(np.arange(c["nrows"]), np.diff(c["rowptr"].astype(np.int64)))
        perm = np.random.default_rng(0).permutation(len(rows))
        t = dg.TripletMatrix(c["nrows"], c["ncols"], rows[perm], c["colids"][perm],
                             c["values"][perm].astype(np.float64))
        b = dg.csr_from_triplets(t, oindex=a.oindex_width, iindex=a.iindex_width,
                                 scalar=a.scalar_width)
        assert b == a


def test_duplicates_and_zeros():
    t = dg.TripletMatrix.from_entries(2, 2, [(0, 1, 1.0), (0, 1, 2.5), (1, 0, 0.0),
                                             (1, 1, -0.0)])
    a = dg.csr_from_triplets(t)
    assert a.values.tolist() == [3.5, 0.0, 0.0] and a.nnz == 3
    assert not np.signbit(a.values[2])  # bincount turns -0.0 into +0.0


def test_width_errors():
    with pytest.raises(EntryOutOfBounds):
        dg.TripletMatrix.from_entries(2, 2, [(2, 0, 1.0)])
    t = dg.TripletMatrix.from_entries(200, 200, [(i, i, 1.0) for i in range(200)])
    with pytest.raises(IndexRangeExceeded):
        dg.csr_from_triplets(t, oindex=8)
    with pytest.raises(IndexRangeExceeded):
        dg.csr_from_triplets(t, iindex=8)
    a = dg.csr_from_triplets(dg.TripletMatrix.from_entries(40010, 40010, [(40000, 40005, 1.0)]))
    with pytest.raises(IndexRangeExceeded):
        dg.to_csr(dg.to_dacsr(a, 16), 16)


def test_validation_and_immutability():
    with pytest.raises(ValueError):
        dg.CsrMatrix(1, 1, np.array([1, 1], np.int32), np.array([0], np.int32), np.array([1.0]))
    with pytest.raises(ValueError):
        dg.CsrMatrix(2, 2, np.array([0, 2, 1], np.int32), np.array([0], np.int32),
                     np.array([1.0]))
    with pytest.raises(ValueError):
        dg.CsrMatrix(1, 3, np.array([0, 2], np.int32), np.array([1, 1], np.int32),
                     np.array([1.0, 2.0]))
    with pytest.raises(ValueError):
        dg.DacsrMatrix(1, 2, np.array([0, 1], np.int32), np.array([2], np.int16),
                       np.array([1.0]))
    v = np.array([1.0])
    a = dg.CsrMatrix(1, 1, np.array([0, 1], np.int32), np.array([0], np.int32), v)
    v[0] = 9.0
    assert a.values[0] == 1.0
    with pytest.raises(ValueError):
        a.values[0] = 2.0


def test_stencil_generators_canonical():
    from paper_2307_06305_b200.workloads import laplacian_2d, laplacian_3d
    for a in (laplacian_2d(17), laplacian_3d(6)):
        b = dg.CsrMatrix(a.nrows, a.ncols, a.rowptr, a.colids, a.values)  # full validation
        assert b == a
        dense = np.zeros((a.nrows, a.ncols))
        rows = np.repeat(np.arange(a.nrows), np.diff(a.rowptr))
        dense[rows, a.colids] = a.values
        assert np.array_equal(dense, dense.T)
    assert laplacian_2d(1024).nnz == 5_238_784 and dg.bandwidth(laplacian_2d(64)) == 64
    assert laplacian_3d(128).nnz == 14_581_760
