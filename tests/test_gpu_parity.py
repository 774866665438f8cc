"""CUDA path vs the CPU oracle (and thereby the reference) — needs a B200.

Bars (tolerances written here, not inferred):
* exact orders (naive/shifted_base/multi_accumulator_3/strip_mined_4 and the
  rowblock/staged/scalar kernels): BIT-EXACT against the reference outputs
  stored in tests/golden/spmv_corpus.npz and against the oracle at full size;
* tree-combining kernels (vector2..warp, rowblock_tree): the reference's own
  verification rule (bench.py:153-157) max|y-ref| <= tol*max(max|ref|,1e-30)
  with tol = 2**-40 (f64) / 1e-5 (f32).
"""

import ctypes

import numpy as np
import pytest
import torch

import oracle
import paper_2307_06305_b200 as dg
from paper_2307_06305_b200 import _native
from paper_2307_06305_b200.device import DeviceMatrix, bandwidth_device, to_dacsr_device
from paper_2307_06305_b200.workloads import laplacian_2d, laplacian_3d, uniform_x
from test_oracle import CORPUS, ORDER_KEYS

pytestmark = pytest.mark.gpu

TREE_VARIANTS = ("vector2", "vector4", "vector8", "vector16", "warp", "rowblock_tree")


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint8)


def within(y, ref):
    tol = 2.0 ** -40 if ref.dtype == np.float64 else 1e-5
    scale = max(float(np.max(np.abs(ref))) if len(ref) else 0.0, 1e-30)
    err = float(np.max(np.abs(y.astype(np.float64) - ref))) if len(ref) else 0.0
    return err <= tol * scale, err / scale


def host_matrix(c, kind):
    if kind == "csr":
        return dg.CsrMatrix(c["nrows"], c["ncols"], c["rowptr"], c["colids"], c["values"])
    return dg.DacsrMatrix(c["nrows"], c["ncols"], c["rowptr"], c["offsets"], c["values"])


@pytest.mark.parametrize("kind", ["csr", "da"])
@pytest.mark.parametrize("variant", list(ORDER_KEYS))
def test_golden_exact_orders_host_api(cuda, kind, variant):
    for k, c in enumerate(CORPUS):
        a = host_matrix(c, kind)
        y = c["y0"].copy()
        out = dg.spmv(a, c["x"], y, c["alpha"], c["beta"], variant)
        assert out is y
        assert np.array_equal(bits(y), bits(c[ORDER_KEYS[variant]])), (k, kind, variant)


@pytest.mark.parametrize("kind", ["csr", "da"])
@pytest.mark.parametrize("variant", ["rowblock", "staged", "scalar", "wstream", "auto"])
def test_golden_exact_kernels_device_api(cuda, kind, variant):
    for k, c in enumerate(CORPUS):
        dm = DeviceMatrix.from_host(host_matrix(c, kind), cuda)
        x = torch.from_numpy(c["x"]).to(cuda)
        y = torch.from_numpy(c["y0"].copy()).to(cuda)
        out = dg.spmv(dm, x, y, c["alpha"], c["beta"], variant)
        assert out is y
        assert np.array_equal(bits(y.cpu().numpy()), bits(c["y_naive"])), (k, kind, variant)


@pytest.mark.parametrize("variant", TREE_VARIANTS)
def test_golden_tree_kernels_within_tolerance(cuda, variant):
    for k, c in enumerate(CORPUS):
        for kind in ("csr", "da"):
            y = c["y0"].copy()
            dg.spmv(host_matrix(c, kind), c["x"], y, c["alpha"], c["beta"], variant)
            ok, rel = within(y, c["y_naive"])
            assert ok, (k, kind, variant, rel)


def test_parallel_row_block_is_inner(cuda):
    for c in CORPUS[:40]:
        a = host_matrix(c, "da")
        for inner in dg.SERIAL_VARIANTS:
            y = c["y0"].copy()
            dg.spmv(a, c["x"], y, c["alpha"], c["beta"], dg.ParallelRowBlock(4, inner))
            assert np.array_equal(bits(y), bits(c[ORDER_KEYS[inner]]))


def test_reference_named_c_abi_entry_points(cuda):
    """dacsr_{csr,da}_{naive,...}_{f64,f32}: the plugin-signature kernels."""
    L = _native.lib()
    names = {"naive": "y_naive", "shifted_base": "y_naive", "multi_acc3": "y_macc3",
             "strip_mined4": "y_strip4"}
    tested = 0
    for c in CORPUS:
        if c["rowptr"].dtype != np.int32 or c["offsets"].dtype != np.int16 or c["nrows"] == 0:
            continue
        if c["alpha"] == 0.0:
            continue  # the alpha==0 short-cut lives in spmv(), not the kernels
        vn = "f64" if c["values"].dtype == np.float64 else "f32"
        dev = {k: torch.from_numpy(np.ascontiguousarray(c[k])).to(cuda)
               for k in ("rowptr", "colids", "offsets", "values", "x")}
        for kind, inner in (("csr", "colids"), ("da", "offsets")):
            for name, key in names.items():
                y = torch.from_numpy(c["y0"].copy()).to(cuda)
                fn = getattr(L, f"dacsr_{kind}_{name}_{vn}")
                rc = fn(dev["rowptr"].data_ptr(), dev[inner].data_ptr() or None,
                        dev["values"].data_ptr() or None, dev["x"].data_ptr() or None,
                        y.data_ptr(), c["alpha"], c["beta"], 0, c["nrows"],
                        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
                assert rc == 0, _native.lib().dacsr_last_error()
                assert np.array_equal(bits(y.cpu().numpy()), bits(c[key])), (kind, name)
                tested += 1
    assert tested > 100


def test_row_range_contract(cuda):
    """Kernels write only [row_start, row_end) (the reference signature)."""
    a = dg.to_dacsr(laplacian_2d(40), 16)
    dm = DeviceMatrix.from_host(a, cuda, plan=False)
    x = torch.from_numpy(uniform_x(a.ncols, 3)).to(cuda)
    for variant in ("staged", "scalar", "vector8"):
        y = torch.full((a.nrows,), 7.0, dtype=torch.float64, device=cuda)
        dm.spmv_into(x, y, 1.0, 0.0, variant, 0, row_start=100, row_end=1000)
        yh = y.cpu().numpy()
        assert (yh[:100] == 7.0).all() and (yh[1000:] == 7.0).all()
        ref = oracle.spmv_kernel("da", a.rowptr, a.colids, a.values, x.cpu().numpy(),
                                 np.full(a.nrows, 7.0), 1.0, 0.0, row_start=100, row_end=1000)
        ok, _ = within(yh, ref)
        assert ok


def _full_parity(a, x, orders=("naive", "multi_accumulator_3", "strip_mined_4")):
    kind = "da" if isinstance(a, dg.DacsrMatrix) else "csr"
    dm = DeviceMatrix.of(a)
    xd = torch.from_numpy(x).to(dm.device)
    for order in orders:
        for alpha, beta in ((1.0, 0.0), (0.7, -0.3)):
            y0 = np.random.default_rng(5).uniform(-1, 1, a.nrows).astype(a.values.dtype)
            yd = torch.from_numpy(y0.copy()).to(dm.device)
            dg.spmv(dm, xd, yd, alpha, beta, order)
            ref = oracle.spmv(kind, a.rowptr, a.colids, a.values, x, y0.copy(), alpha, beta,
                              order=order, threads=8)
            assert np.array_equal(bits(yd.cpu().numpy()), bits(ref)), (kind, order, alpha)
    return dm


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_config_c1_c2_full_size_bit_exact(cuda, dtype):
    for builder, nx in ((laplacian_2d, 1024), (laplacian_3d, 128)):
        csr = builder(nx, dtype=dtype)
        x = uniform_x(csr.ncols, seed=11).astype(dtype)
        _full_parity(csr, x, orders=("naive",))
        _full_parity(dg.to_dacsr(csr, 16), x)


def test_skewed_long_rows_bit_exact(cuda):  # noqa: C901
    """C4-like skew: rows of 1000-4096 entries among 5-entry rows; the
    cooperative long-row path keeps every exact order bit-exact."""
    from paper_2307_06305_b200.workloads import add_skew_rows
    base = laplacian_2d(256)
    a = add_skew_rows(base, frac=0.01, alpha=1.5, cap=4096, band=1024, seed=3)
    # plus a handful of guaranteed long rows (Pareto tails are rare at this n)
    a = add_skew_rows(a, frac=12 / a.nrows, alpha=0.05, cap=2000, band=1024, seed=4)
    assert np.diff(a.rowptr).max() > 1000
    x = uniform_x(a.ncols, seed=4)
    _full_parity(a, x)
    _full_parity(dg.to_dacsr(a, 16), x)
    d = dg.to_dacsr(a, 16)
    ref = oracle.spmv("da", a.rowptr, d.colids, a.values, x)
    for kernel in ("rowblock", "staged", "wstream"):
        y = dg.spmv(d, x, variant=kernel)
        assert np.array_equal(y.view(np.uint64), ref.view(np.uint64)), kernel
    # the warp-stream window pinned small (most chunks go to the side CTAs)
    # and large (none do)
    dm = DeviceMatrix.from_host(d, cuda)
    xd = torch.from_numpy(x).to(cuda)
    for rows in (32, 64):
        for vcap in (64, 96, 160, 1024, 4096):
            dm.set_chunk_window(vcap, rows)
            y = dg.spmv(dm, xd, variant="wstream")
            assert np.array_equal(bits(y.cpu().numpy()), bits(ref)), (vcap, rows)
    for variant in ("rowblock_tree", "vector8", "warp"):
        y = dg.spmv(dg.to_dacsr(a, 16), x, variant=variant)
        ref = oracle.spmv("da", a.rowptr, dg.to_dacsr(a, 16).colids, a.values, x)
        assert within(y, ref)[0], variant


def test_device_conversion_matches_host(cuda):
    csr = laplacian_3d(40)
    dm = DeviceMatrix.from_host(csr, cuda)
    assert bandwidth_device(dm) == dg.bandwidth(csr)
    dd = to_dacsr_device(dm, 16)
    assert np.array_equal(dd.colids.cpu().numpy(), dg.to_dacsr(csr, 16).colids)
    with pytest.raises(dg.errors.BandwidthExceedsIndexRange):
        to_dacsr_device(dm, 8)


def test_sumsq_chunks_deterministic(cuda):
    from paper_2307_06305_b200.power import chunked_sumsq
    y = torch.randn(1 << 20, dtype=torch.float64, device=cuda)
    a = chunked_sumsq(y, 1 << 14)
    b = chunked_sumsq(y, 1 << 14)
    assert a == b
    assert abs(a - float((y * y).sum())) <= 1e-12 * a


def test_widths_int64_rowptr_int8_offsets_int64_colids(cuda):
    """Every device layout the library instantiates, against the oracle."""
    from paper_2307_06305_b200.core import _trusted
    base = laplacian_2d(100)                       # bandwidth 100: fits int8 offsets
    x = uniform_x(base.ncols, seed=8)
    for vdt in (np.float64, np.float32):
        vals = base.values.astype(vdt)
        xv = x.astype(vdt)
        for rp_dt in (np.int32, np.int64):
            rp = base.rowptr.astype(rp_dt)
            mats = [
                _trusted(dg.CsrMatrix, base.nrows, base.ncols, rp, base.colids.astype(np.int32), vals),
                _trusted(dg.DacsrMatrix, base.nrows, base.ncols, rp,
                         dg.to_dacsr(base, 8).colids, vals),
                _trusted(dg.DacsrMatrix, base.nrows, base.ncols, rp,
                         dg.to_dacsr(base, 16).colids, vals),
                _trusted(dg.DacsrMatrix, base.nrows, base.ncols, rp,
                         dg.to_dacsr(base, 32).colids, vals),
            ]
            for a in mats:
                dm = DeviceMatrix.from_host(a, cuda)
                if a.rowptr.dtype == np.int64:    # keep the int64 rowptr on device
                    dm = DeviceMatrix(dm.kind, a.nrows, a.ncols,
                                      torch.from_numpy(a.rowptr).to(cuda), dm.colids, dm.values)
                kind = "da" if isinstance(a, dg.DacsrMatrix) else "csr"
                ref = oracle.spmv(kind, a.rowptr, a.colids, a.values, xv)
                for variant in ("naive", "wstream", "rowblock", "staged", "scalar"):
                    y = dg.spmv(dm, torch.from_numpy(xv).to(cuda), variant=variant)
                    assert np.array_equal(bits(y.cpu().numpy()), bits(ref)), (kind, variant,
                                                                              rp_dt, vdt)


def test_wstream_empty_rows_and_chunks(cuda):
    """Empty rows, whole empty 32/64-row chunks, and an empty tail."""
    rng = np.random.default_rng(12)
    n = 5000
    counts = rng.integers(0, 6, n)
    counts[100:300] = 0          # empty chunks
    counts[-200:] = 0            # empty tail
    rp = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    cols = np.concatenate([np.sort(rng.choice(np.arange(max(0, r - 40), min(n, r + 41)),
                                              size=k, replace=False))
                           for r, k in enumerate(counts)]).astype(np.int32)
    a = dg.CsrMatrix(n, n, rp, cols, rng.standard_normal(len(cols)))
    d = dg.to_dacsr(a, 16)
    x = uniform_x(n, 3)
    ref = oracle.spmv("da", d.rowptr, d.colids, d.values, x)
    dm = DeviceMatrix.from_host(d, cuda)
    xd = torch.from_numpy(x).to(cuda)
    for rows in (32, 64):
        for vcap in (64, 128, 512):
            dm.set_chunk_window(vcap, rows)
            y = dg.spmv(dm, xd, variant="wstream")
            assert np.array_equal(bits(y.cpu().numpy()), bits(ref)), (rows, vcap)


def test_streamed_host_path_bit_exact(cuda):
    """spmv(A, x_host, y_host) above STREAMED_MIN_ROWS pipelines the copies
    by row pieces; results equal the device path bit for bit (pinned and
    pageable host buffers, beta = 0 and beta != 0, DA and CSR)."""
    from paper_2307_06305_b200.spmv import STREAMED_MIN_ROWS
    csr = laplacian_2d(640)                       # 409,600 rows >= 2^18
    assert csr.nrows >= STREAMED_MIN_ROWS
    x = uniform_x(csr.ncols, 5)
    y0 = np.random.default_rng(6).uniform(-1, 1, csr.nrows)
    for a in (dg.to_dacsr(csr, 16), csr):
        kind = "da" if isinstance(a, dg.DacsrMatrix) else "csr"
        for alpha, beta in ((1.0, 0.0), (0.5, -2.0)):
            ref = oracle.spmv(kind, a.rowptr, a.colids, a.values, x, y0.copy(), alpha, beta)
            y = y0.copy()
            dg.spmv(a, x, y, alpha, beta)
            assert np.array_equal(bits(y), bits(ref)), (kind, beta)
            xp = torch.empty(len(x), dtype=torch.float64, pin_memory=True)
            yp = torch.empty(len(y0), dtype=torch.float64, pin_memory=True)
            xp.numpy()[:] = x
            yp.numpy()[:] = y0
            out = dg.spmv(a, xp.numpy(), yp.numpy(), alpha, beta)
            assert np.array_equal(bits(out), bits(ref)), (kind, beta, "pinned")
