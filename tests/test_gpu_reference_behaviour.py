"""The reference's operator tests (/root/reference/pkg/tests/test_spmv.py),
restated against this package on the GPU: the same calls must give the same
results and the same exceptions (drop-in check)."""

import numpy as np
import pytest

import oracle
import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.errors import DimensionMismatch, UnsupportedScalarWidth

pytestmark = pytest.mark.gpu

SAMPLE = [(0, 0, 1.0), (1, 2, 2.0), (2, 1, 3.0), (2, 3, 4.0), (3, 3, 5.0)]


def entries_matrix(nrows, ncols, entries, oindex=32, iindex=32, scalar=64):
    t = dg.TripletMatrix.from_entries(nrows, ncols, entries)
    return dg.csr_from_triplets(t, oindex=oindex, iindex=iindex, scalar=scalar)


def dense_of(a):
    d = np.zeros((a.nrows, a.ncols))
    for r in range(a.nrows):
        for i in range(int(a.rowptr[r]), int(a.rowptr[r + 1])):
            c = int(a.colids[i]) + (r if isinstance(a, dg.DacsrMatrix) else 0)
            d[r, c] += float(a.values[i])
    return d


def dense_matvec(d, x, y0=None, alpha=1.0, beta=0.0):
    y = np.zeros(d.shape[0])
    for r in range(d.shape[0]):
        acc = 0.0
        for c in range(d.shape[1]):
            acc += float(d[r, c]) * float(x[c])
        y[r] = alpha * acc + (beta * float(y0[r]) if beta != 0.0 else 0.0)
    return y


@pytest.fixture
def sample():
    return entries_matrix(4, 4, SAMPLE)


def both(a, bits=16):
    return [a, dg.to_dacsr(a, bits)]


def test_sample_all_ones_and_beta(cuda, sample):
    for m in both(sample):
        assert dg.spmv(m, np.ones(4)).tolist() == [1.0, 2.0, 7.0, 5.0]
        y = np.ones(4)
        assert dg.spmv(m, np.ones(4), y, alpha=1.0, beta=2.0).tolist() == [3.0, 4.0, 9.0, 7.0]


def test_alpha_zero_beta_one_is_identity(cuda, sample):
    y0 = np.array([0.25, -1.5, 3.0, 7.5])
    for m in both(sample):
        y = y0.copy()
        out = dg.spmv(m, np.ones(4), y, alpha=0.0, beta=1.0)
        assert out is y and np.array_equal(y, y0)


def test_alpha_zero_scales_and_zeroes(cuda, sample):
    y0 = np.array([0.25, -1.5, np.nan, 7.5], dtype=np.float32)
    a32 = entries_matrix(4, 4, SAMPLE, scalar=32)
    for m in both(a32):
        y = y0.copy()
        dg.spmv(m, np.ones(4, np.float32), y, alpha=0.0, beta=-3.0)
        want = (np.float64(-3.0) * y0).astype(np.float32)   # reference 150-156
        assert np.array_equal(y, want, equal_nan=True)
        y = y0.copy()
        dg.spmv(m, np.ones(4, np.float32), y, alpha=0.0, beta=0.0)
        assert y.tolist() == [0.0] * 4


def test_identity_scaling_and_nan_safety(cuda):
    a = entries_matrix(5, 5, [(i, i, 1.0) for i in range(5)])
    x = np.arange(1.0, 6.0)
    for m in both(a):
        assert np.array_equal(dg.spmv(m, x, alpha=2.0), 2.0 * x)
        for variant in dg.SERIAL_VARIANTS + ("auto", "vector8"):
            y = np.full(5, np.nan)
            dg.spmv(m, x, y, beta=0.0, variant=variant)
            assert not np.isnan(y).any()


def test_empty_rows_rectangular_and_empty(cuda):
    a = entries_matrix(3, 3, [(1, 1, 4.0)])
    y = np.ones(3)
    dg.spmv(a, np.ones(3), y, alpha=1.0, beta=3.0)
    assert y.tolist() == [3.0, 7.0, 3.0]
    tall = entries_matrix(6, 3, [(0, 0, 1.0), (1, 1, 2.0), (2, 2, 3.0), (2, 0, 4.0)])
    wide = entries_matrix(2, 7, [(0, 6, 1.0), (1, 0, 2.0)])
    for mat, x in ((tall, np.ones(3)), (wide, np.arange(1.0, 8.0))):
        want = dense_matvec(dense_of(mat), x)
        for m in both(mat):
            for variant in dg.SERIAL_VARIANTS:
                assert np.array_equal(dg.spmv(m, x, variant=variant), want)
    assert dg.spmv(entries_matrix(0, 0, []), np.empty(0)).shape == (0,)
    out = dg.spmv(a, np.ones(3))
    assert out.dtype == np.float64 and out.shape == (3,)


def test_validation_errors(cuda, sample):
    with pytest.raises(DimensionMismatch):
        dg.spmv(sample, np.ones(3))
    with pytest.raises(DimensionMismatch):
        dg.spmv(sample, np.ones(4), np.ones(5))
    with pytest.raises(UnsupportedScalarWidth):
        dg.spmv(sample, np.ones(4, np.float32))
    with pytest.raises(ValueError):
        dg.spmv(sample, np.ones(4), variant="vectorized")
    with pytest.raises(ValueError):
        dg.spmv(sample, np.ones(4), y=None, beta=1.0)


def test_dense_oracle_f64_f32_and_bit_exact_csr_da(cuda):
    rng = np.random.default_rng(23)
    for trial in range(30):
        nr, nc = int(rng.integers(1, 128)), int(rng.integers(1, 128))
        t = int(round(0.1 * nr * nc))
        ent = list(zip(rng.integers(0, nr, t).tolist(), rng.integers(0, nc, t).tolist(),
                       rng.uniform(0.5, 1.5, t).tolist()))
        scalar = 32 if trial % 3 == 2 else 64
        a = entries_matrix(nr, nc, ent, scalar=scalar)
        sd = a.values.dtype
        x = rng.uniform(0.5, 1.5, nc).astype(sd)
        y0 = rng.uniform(-1.0, 1.0, nr).astype(sd)
        alpha, beta = [(1.0, 0.0), (2.0, 0.5), (0.7, -0.3)][trial % 3]
        want = dense_matvec(dense_of(a), x, y0, alpha, beta)
        tol = 1e-12 if sd == np.float64 else 1e-5
        res = []
        for m in both(a):
            for variant in dg.SERIAL_VARIANTS + tuple(dg.ParallelRowBlock(k, "naive") for k in (2, 8)):
                y = y0.copy()
                dg.spmv(m, x, y, alpha, beta, variant)
                scale = max(np.abs(want).max(), 1e-300)
                assert np.abs(y.astype(np.float64) - want).max() / scale <= tol
                if variant == "naive":
                    res.append(y)
        assert np.array_equal(res[0], res[1])          # naive CSR == naive DA bit-exact
        kind_ref = oracle.spmv("csr", a.rowptr, a.colids, a.values, x, y0.copy(), alpha, beta)
        assert np.array_equal(res[0], kind_ref)


def test_narrow_index_widths(cuda):
    e = [(0, 0, 1.0), (1, 0, 2.0), (1, 2, 3.0), (3, 3, 4.0)]
    a = entries_matrix(4, 4, e, oindex=8, iindex=8)
    d = dg.to_dacsr(a, 8)
    x = np.array([1.0, 2.0, 3.0, 4.0])
    want = dense_matvec(dense_of(a), x)
    assert np.array_equal(dg.spmv(a, x), want) and np.array_equal(dg.spmv(d, x), want)


def test_host_arrays_on_a_caller_stream(cuda):
    """Host x / y with a non-default stream: the copies and the kernel are
    ordered on that stream, pinned and pageable y alike; the
    stream is kept busy first so a missing dependency would show."""
    import torch
    from paper_2307_06305_b200.workloads import laplacian_2d, uniform_x
    a = dg.to_dacsr(laplacian_2d(300), 16)
    x = uniform_x(a.ncols, 4)
    y0 = np.random.default_rng(5).uniform(-1, 1, a.nrows)
    want = oracle.spmv("da", a.rowptr, a.colids, a.values, x, y0.copy(), 0.5, 2.0)
    s = torch.cuda.Stream()
    busy = torch.ones(1 << 24, device=cuda)
    for pinned in (False, True):
        with torch.cuda.stream(s):
            for _ in range(20):
                busy.mul_(1.0000001)  # a backlog on the stream before the call
        if pinned:
            y = torch.from_numpy(y0.copy()).pin_memory().numpy()
        else:
            y = y0.copy()
        out = dg.spmv(a, x, y, 0.5, 2.0, stream=s)
        assert out is y
        s.synchronize()
        assert np.array_equal(y, want), pinned
