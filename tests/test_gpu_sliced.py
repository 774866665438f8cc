"""The sliced device layout (dacsr_slices_t) and its SpMV kernel — needs a B200.

The layout is a bit-for-bit re-arrangement of the CSR/DA-CSR entries
(32-row slices, entry j of lane l at slice_ptr[s] + 32*j + l); the kernel
folds each row in the reference's naive order, so every result here is
BIT-EXACT against the reference outputs (tests/golden) and the oracle.
Spill rows (longer than the layout's max_len) take the CSR path inside the
same launch; forcing small max_len values exercises it everywhere.
"""

import numpy as np
import pytest
import torch

import oracle
import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.workloads import add_skew_rows, laplacian_2d, laplacian_3d, uniform_x
from test_gpu_parity import bits, host_matrix
from test_oracle import CORPUS

pytestmark = pytest.mark.gpu


def unslice(dm):
    """Rebuild {row: (inner, values)} from the main and medium slices, and
    return the medium / long row lists."""
    _, sl, t = dm._sliced
    n = dm.row_end - dm.row_start
    lens = t["row_len"].cpu().numpy()[:n].astype(np.int64)
    rows = {}
    ptr = t["slice_ptr"].cpu().numpy()
    inn, val = t["inner"].cpu().numpy(), t["values"].cpu().numpy()
    for r in range(n):
        if lens[r] <= sl.max_len:
            s_, lane = divmod(r, 32)
            slots = ptr[s_] + 32 * np.arange(lens[r]) + lane
            rows[r] = (inn[slots], val[slots])
    medium = t["medium_rows"].cpu().numpy()[:sl.n_medium]
    if sl.n_medium:
        mptr = t["m_slice_ptr"].cpu().numpy()
        minn, mval = t["m_inner"].cpu().numpy(), t["m_values"].cpu().numpy()
        for k, r in enumerate(medium):
            m_, lane = divmod(k, 32)
            slots = mptr[m_] + 32 * np.arange(lens[r - dm.row_start]) + lane
            rows[int(r)] = (minn[slots], mval[slots])
    return rows, medium, t["long_rows"].cpu().numpy()[:sl.n_long]


@pytest.mark.parametrize("kind", ["csr", "da"])
def test_layout_is_a_rearrangement(cuda, kind):
    for c in CORPUS[::7]:
        a = host_matrix(c, kind)
        dm = DeviceMatrix.from_host(a, cuda)
        for max_len, medium_len in ((1, 1), (1, 3), (2, 254), (254, 254)):
            dm.build_slices(max_len, medium_len)
            rows, medium, long_ = unslice(dm)
            rp = np.asarray(a.rowptr, dtype=np.int64)
            lens = np.diff(rp)
            medium_len = max(max_len, medium_len)
            assert list(medium) == [r for r in range(a.nrows) if max_len < lens[r] <= medium_len]
            assert list(long_) == [r for r in range(a.nrows) if lens[r] > medium_len]
            assert sorted(rows) == [r for r in range(a.nrows) if lens[r] <= medium_len]
            for r, (inn, val) in rows.items():
                b, e = rp[r], rp[r + 1]
                assert np.array_equal(inn, np.asarray(a.colids)[b:e].astype(inn.dtype))
                assert np.array_equal(bits(val), bits(np.asarray(a.values)[b:e]))


@pytest.mark.parametrize("kind", ["csr", "da"])
@pytest.mark.parametrize("lens", [None, (1, 1), (1, 3), (3, 40)])
@pytest.mark.parametrize("variant", ["sliced", "sliced_pipe", "tiled"])
def test_golden_bit_exact(cuda, kind, lens, variant):
    max_len = lens
    for k, c in enumerate(CORPUS):
        dm = DeviceMatrix.from_host(host_matrix(c, kind), cuda)
        if lens is not None:
            dm.build_slices(*lens)
        x = torch.from_numpy(c["x"]).to(cuda)
        y = torch.from_numpy(c["y0"].copy()).to(cuda)
        out = dg.spmv(dm, x, y, c["alpha"], c["beta"], variant)
        assert out is y
        assert np.array_equal(bits(y.cpu().numpy()), bits(c["y_naive"])), (k, kind, max_len)


@pytest.mark.parametrize("variant", ["sliced", "sliced_pipe", "tiled"])
def test_row_ranges_and_x_offset(cuda, variant):
    a = dg.to_dacsr(add_skew_rows(laplacian_2d(96), frac=0.03, alpha=0.3, cap=700, band=500,
                                  seed=4), 16)
    dm = DeviceMatrix.from_host(a, cuda)
    dm.build_slices(6, 40)
    info = dm.slices_info()
    assert info["n_medium"] > 0 and info["n_long"] > 0
    xh = uniform_x(a.ncols, 9)
    pad = 37
    x_ext = torch.zeros(a.ncols + 2 * pad, dtype=torch.float64, device=cuda)
    x_ext[pad:pad + a.ncols] = torch.from_numpy(xh).to(cuda)
    rng = np.random.default_rng(3)
    for _ in range(12):
        r0, r1 = sorted(int(v) for v in rng.integers(0, a.nrows + 1, 2))
        y = torch.full((a.nrows,), 5.0, dtype=torch.float64, device=cuda)
        dm.spmv_into(x_ext, y, 0.5, 0.0, variant, 0, x_offset=pad, row_start=r0, row_end=r1)
        ref = oracle.spmv_kernel("da", a.rowptr, a.colids, a.values, xh, np.full(a.nrows, 5.0),
                                 0.5, 0.0, row_start=r0, row_end=r1)
        assert np.array_equal(bits(y.cpu().numpy()), bits(ref)), (r0, r1)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.bfloat16, torch.float16])
def test_c2_full_size_matches_exact_kernels(cuda, dtype):
    a = dg.to_dacsr(laplacian_3d(128), 16)
    dm = DeviceMatrix.of(a).astype(dtype)
    x = torch.from_numpy(uniform_x(a.ncols, 1)).to(cuda).to(dtype)
    want = dm.spmv_into(x, torch.empty(a.nrows, dtype=dtype, device=cuda), 1.0, 0.0, "wstream")
    got = dm.spmv_into(x, torch.empty(a.nrows, dtype=dtype, device=cuda), 1.0, 0.0, "sliced")
    got5 = dm.spmv_into(x, torch.empty(a.nrows, dtype=dtype, device=cuda), 1.0, 0.0,
                        "sliced_pipe")
    got6 = dm.spmv_into(x, torch.empty(a.nrows, dtype=dtype, device=cuda), 1.0, 0.0, "tiled")
    as_int = {8: torch.int64, 4: torch.int32, 2: torch.int16}[dtype.itemsize]
    assert torch.equal(got.view(as_int), want.view(as_int))
    assert torch.equal(got5.view(as_int), want.view(as_int))
    assert torch.equal(got6.view(as_int), want.view(as_int))
    if dtype == torch.float64:
        ref = oracle.spmv("da", a.rowptr, a.colids, a.values, x.cpu().numpy())
        assert np.array_equal(bits(got.cpu().numpy()), bits(ref))


def test_skewed_spill_rows_full_size(cuda):
    """C4-like: 1% Pareto rows (up to ~3000 entries) spill; warp-folded."""
    a = dg.to_dacsr(add_skew_rows(laplacian_2d(1024), frac=0.01, alpha=1.5, cap=3000, band=1000,
                                  seed=7), 16)
    dm = DeviceMatrix.of(a)
    x = torch.from_numpy(uniform_x(a.ncols, 2)).to(cuda)
    ref = oracle.spmv("da", a.rowptr, a.colids, a.values, x.cpu().numpy())
    for variant in ("sliced", "sliced_pipe", "tiled"):
        got = dm.spmv_into(x, torch.empty(a.nrows, dtype=torch.float64, device=cuda), 1.0, 0.0,
                           variant)
        assert np.array_equal(bits(got.cpu().numpy()), bits(ref)), variant
    info = dm.slices_info()
    assert info["n_medium"] > 0 and info["n_long"] > 0


@pytest.mark.parametrize("variant", ["sliced", "sliced_pipe", "tiled"])
def test_streamed_host_path_on_slices(cuda, variant):
    """spmv(A, x_host, y_host) with the slices: the row pieces of the
    streamed host path share the whole matrix's layout; bit-exact."""
    a = dg.to_dacsr(add_skew_rows(laplacian_2d(512), frac=0.01, alpha=1.5, cap=600, band=500,
                                  seed=3), 16)
    dm = DeviceMatrix.of(a)
    dm.build_slices(5, 32)
    dm.tuned_kernel = variant
    x = uniform_x(a.ncols, 4)
    yp = torch.empty(a.nrows, dtype=torch.float64, pin_memory=True)
    for alpha, beta in ((1.0, 0.0), (0.5, -2.0)):
        y0 = np.random.default_rng(1).uniform(-1, 1, a.nrows)
        ref = oracle.spmv("da", a.rowptr, a.colids, a.values, x, y0.copy(), alpha, beta)
        y = y0.copy()                      # pageable: y through the device + D2H
        dg.spmv(a, x, y, alpha, beta)
        assert np.array_equal(bits(y), bits(ref)), (alpha, beta)
        yp.numpy()[:] = y0                 # pinned: the kernels store y in host memory
        dg.spmv(a, x, yp.numpy(), alpha, beta)
        assert np.array_equal(bits(yp.numpy()), bits(ref)), (alpha, beta, "pinned")
    dm.tuned_kernel = None


def test_l2_prefetch_flag_keeps_bits(cuda):
    """dacsr_plan_t.flags (no L2 bulk prefetch) changes timing only."""
    a = dg.to_dacsr(add_skew_rows(laplacian_2d(256), frac=0.02, alpha=1.2, cap=400, band=200,
                                  seed=8), 16)
    dm = DeviceMatrix.from_host(a, cuda)
    dm.build_slices()
    x = torch.from_numpy(uniform_x(a.ncols, 3)).to(cuda)
    ref = oracle.spmv("da", a.rowptr, a.colids, a.values, x.cpu().numpy())
    for on in (False, True):
        dm.set_sliced_l2_prefetch(on)
        for variant in ("sliced", "sliced_pipe"):
            y = dm.spmv_into(x, torch.empty(a.nrows, dtype=torch.float64, device=cuda), 1.0,
                             0.0, variant)
            assert np.array_equal(bits(y.cpu().numpy()), bits(ref)), (on, variant)


def test_autotune_then_exact(cuda):
    """autotune() (kernel, slice width, L2-prefetch flag, dropping an unused
    sliced copy) only changes speed: 'naive' stays bit-exact afterwards."""
    cases = [c for c in CORPUS if c["nrows"] >= 64][:6]
    cases.append(None)  # a skewed matrix with medium and long rows
    for c in cases:
        if c is None:
            a = dg.to_dacsr(add_skew_rows(laplacian_2d(128), frac=0.02, alpha=1.2, cap=500,
                                          band=300, seed=5), 16)
            x_h = uniform_x(a.ncols, 6)
            y0 = np.zeros(a.nrows)
            alpha, beta, want = 1.0, 0.0, None
        else:
            a = host_matrix(c, "da")
            x_h, y0, alpha, beta, want = c["x"], c["y0"], c["alpha"], c["beta"], c["y_naive"]
        dm = DeviceMatrix.from_host(a, cuda)
        x = torch.from_numpy(np.ascontiguousarray(x_h)).to(cuda)
        for cold in (False, True):
            dm.autotune(cold=cold, x=x, reps=2)
            assert dm.tuned_kernel in dg.GPU_VARIANTS
            y = torch.from_numpy(np.ascontiguousarray(y0).copy()).to(cuda)
            dg.spmv(dm, x, y, alpha, beta, "naive")
            ref = want if want is not None else oracle.spmv(
                "da", a.rowptr, a.colids, a.values, np.asarray(x_h), np.asarray(y0).copy(),
                alpha, beta)
            assert np.array_equal(bits(y.cpu().numpy()), bits(ref)), (dm.tuned_kernel, cold)
