"""Host-side semantics of the operator API that hold before any device work
(mirrors the reference's validation, spmv/__init__.py:104-183)."""

import json
import os

import numpy as np
import pytest

import paper_2307_06305_b200 as dg
from conftest import GOLDEN
from paper_2307_06305_b200.errors import DimensionMismatch, UnsupportedScalarWidth

SAMPLE = [(0, 0, 1.0), (1, 2, 2.0), (2, 1, 3.0), (2, 3, 4.0), (3, 3, 5.0)]


@pytest.fixture
def sample():
    return dg.csr_from_triplets(dg.TripletMatrix.from_entries(4, 4, SAMPLE))


def test_sample_layout(sample):
    assert sample.rowptr.tolist() == [0, 1, 2, 4, 5]
    assert sample.colids.tolist() == [0, 2, 1, 3, 3]
    d = dg.to_dacsr(sample, 16)
    assert d.colids.tolist() == [0, 1, -1, 1, 0] and d.colids.dtype == np.int16
    assert d.rowptr is sample.rowptr or np.array_equal(d.rowptr, sample.rowptr)


def test_type_and_shape_errors(sample):
    with pytest.raises(TypeError):
        dg.spmv("not a matrix", np.ones(4))
    with pytest.raises(DimensionMismatch):
        dg.spmv(sample, np.ones(3))
    with pytest.raises(DimensionMismatch):
        dg.spmv(sample, np.ones(4), np.ones(5))
    with pytest.raises(ValueError):
        dg.spmv(sample, np.ones(4), None, beta=1.0)
    with pytest.raises(TypeError):
        dg.spmv(sample, np.ones(4), [0.0] * 4, beta=1.0)


def test_scalar_width_errors(sample):
    with pytest.raises(UnsupportedScalarWidth):
        dg.spmv(sample, np.ones(4, np.float32))
    with pytest.raises(UnsupportedScalarWidth):
        dg.spmv(sample, np.ones(4), np.ones(4, np.float32))
    with pytest.raises(UnsupportedScalarWidth):
        dg.spmv(sample, np.ones(4, np.float16), np.ones(4, np.float16))


def test_variant_and_backend_errors(sample):
    with pytest.raises(ValueError):
        dg.spmv(sample, np.ones(4), variant="vectorized")
    with pytest.raises(ValueError):
        dg.spmv(sample, np.ones(4), backend="numba")
    with pytest.raises(ValueError):
        dg.ParallelRowBlock(0, "naive")
    with pytest.raises(ValueError):
        dg.ParallelRowBlock(2, "bogus")
    with pytest.raises(ValueError):
        dg.ParallelRowBlock(2, dg.ParallelRowBlock(2, "naive"))


def test_backend_env(monkeypatch):
    assert dg.available_backends() == ("cuda",)
    monkeypatch.setenv("DACSR_BACKEND", "numpy")
    with pytest.raises(ValueError):
        dg.default_backend()
    monkeypatch.setenv("DACSR_BACKEND", "cuda")
    assert dg.default_backend() == "cuda"


def test_variant_mapping():
    from paper_2307_06305_b200.spmv import resolve_variant
    assert resolve_variant("naive") == ("exact", 0)
    assert resolve_variant("shifted_base") == ("exact", 0)
    assert resolve_variant("multi_accumulator_3") == ("exact", 1)
    assert resolve_variant("strip_mined_4") == ("exact", 2)
    assert resolve_variant(dg.ParallelRowBlock(8, "strip_mined_4")) == ("exact", 2)
    assert resolve_variant("vector8") == ("vector8", 3)


def test_row_blocks_golden():
    with open(os.path.join(GOLDEN, "row_blocks.json")) as f:
        for c in json.load(f):
            got = dg.row_blocks(np.array(c["rowptr"], np.int64), c["k"])
            assert [list(b) for b in got] == c["cuts"]


def test_work_flops(sample):
    assert dg.work_flops(sample) == 2 * 5 + 2 * 4
    assert dg.work_flops(nnz=127_729_899, nrows=2_911_419) == 261_282_636
