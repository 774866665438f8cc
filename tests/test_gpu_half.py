"""16-bit values on the GPU (DeviceMatrix.astype: binary16 / bfloat16
values, x and y) against the CPU oracle — needs a B200.

Bar: BIT-EXACT for the exact orders (the products are exact and the f64 sum
follows the oracle's order; one RNE rounding on the store), the reference's
verification rule for the tree kernels with tol = 2^-8 (binary16) / 2^-5
(bfloat16) relative to max|ref| — those only differ by the sum order before
the 16-bit rounding, so at most one unit in the last place of the result
scale.  See tests/test_oracle_half.py for the oracle's own pin.
"""

import numpy as np
import pytest
import torch

import oracle
import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.errors import UnsupportedScalarWidth
from paper_2307_06305_b200.workloads import add_skew_rows, laplacian_2d, laplacian_3d

pytestmark = pytest.mark.gpu

DTYPES = {"float16": torch.float16, "bfloat16": torch.bfloat16}


def host_bits(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def oracle_y(kind, dm16, x16, y16, alpha, beta, order):
    bf16 = dm16.values.dtype == torch.bfloat16
    rp = dm16.rowptr.cpu().numpy()
    ci = dm16.colids.cpu().numpy()
    v, x, y = host_bits(dm16.values), host_bits(x16), host_bits(y16).copy()
    if bf16:
        oracle.spmv_kernel(kind, rp, ci, v, x, y, alpha, beta, order, bf16=True)
        return y
    yh = y.view(np.float16)
    oracle.spmv_kernel(kind, rp, ci, v.view(np.float16), x.view(np.float16), yh, alpha, beta,
                       order)
    return yh.view(np.uint16)


def matrices():
    base = laplacian_2d(96)
    skew = add_skew_rows(base, frac=0.01, alpha=1.5, cap=3000, band=400, seed=3)
    skew = add_skew_rows(skew, frac=8 / skew.nrows, alpha=0.05, cap=1500, band=400, seed=4)
    return {"lap3d": laplacian_3d(20), "skew": skew}


@pytest.mark.parametrize("dtype", list(DTYPES))
def test_half_exact_kernels_bit_exact(cuda, dtype):
    g = torch.Generator(device="cpu").manual_seed(5)
    for name, csr in matrices().items():
        vals = torch.randn(csr.nnz, generator=g, dtype=torch.float64)
        csr = dg.CsrMatrix(csr.nrows, csr.ncols, csr.rowptr, csr.colids, vals.numpy())
        cases = [("csr", csr), ("da", dg.to_dacsr(csr, 16))]
        if dg.bandwidth(csr) <= 127:
            cases.append(("da", dg.to_dacsr(csr, 8)))
        for kind, a in cases:
            dm = DeviceMatrix.from_host(a, cuda).astype(DTYPES[dtype])
            x = torch.randn(a.ncols, generator=g, dtype=torch.float64).to(cuda).to(DTYPES[dtype])
            y0 = torch.randn(a.nrows, generator=g, dtype=torch.float64).to(cuda).to(DTYPES[dtype])
            for alpha, beta in [(1.0, 0.0), (0.7, -0.3), (2.0, 1.0)]:
                for order in ("naive", "multi_accumulator_3", "strip_mined_4"):
                    ref = oracle_y(kind, dm, x, y0, alpha, beta, order)
                    kernels = (["wstream", "rowblock", "scalar", "staged", "auto"]
                               if order == "naive" else [order])
                    for k in kernels:
                        y = y0.clone()
                        if k == order:
                            out = dg.spmv(dm, x, y, alpha, beta, order)
                        else:
                            out = dg.spmv(dm, x, y, alpha, beta, k)
                        assert out is y
                        assert np.array_equal(host_bits(y), ref), (name, kind, dtype, k, order,
                                                                   alpha, beta)


@pytest.mark.parametrize("dtype", list(DTYPES))
def test_half_beta_zero_never_reads_y_and_alpha_zero(cuda, dtype):
    a = dg.to_dacsr(laplacian_2d(64), 16)
    dm = DeviceMatrix.from_host(a, cuda).astype(dtype)
    x = torch.ones(a.ncols, dtype=DTYPES[dtype], device=cuda)
    y = torch.full((a.nrows,), float("nan"), dtype=DTYPES[dtype], device=cuda)
    dg.spmv(dm, x, y, 1.0, 0.0)
    assert not torch.isnan(y).any()
    ref = oracle_y("da", dm, x, torch.zeros_like(y), 1.0, 0.0, "naive")
    assert np.array_equal(host_bits(y), ref)
    y2 = y.clone()
    dg.spmv(dm, x, y2, 0.0, 2.0)  # alpha == 0: y <- beta*y, matrix untouched
    assert torch.equal(y2, (y.double() * 2.0).to(DTYPES[dtype]))


@pytest.mark.parametrize("dtype", list(DTYPES))
def test_half_tree_kernels_within_tolerance(cuda, dtype):
    tol = 2.0 ** -8 if dtype == "float16" else 2.0 ** -5
    csr = matrices()["skew"]
    a = dg.to_dacsr(csr, 16)
    dm = DeviceMatrix.from_host(a, cuda).astype(dtype)
    x = torch.rand(a.ncols, dtype=torch.float64, device=cuda).to(DTYPES[dtype])
    ref = oracle.from_half_bits(oracle_y("da", dm, x, torch.zeros(a.nrows, dtype=DTYPES[dtype]),
                                         1.0, 0.0, "naive"), dtype == "bfloat16")
    for variant in ("vector2", "vector8", "vector16", "warp", "rowblock_tree"):
        y = dg.spmv(dm, x, None, variant=variant).double().cpu().numpy()
        scale = max(np.abs(ref).max(), 1e-30)
        assert np.abs(y - ref).max() <= tol * scale, variant


def test_half_widths_rejected_on_host_matrices(cuda):
    """Reference behaviour kept: host matrices stay f32/f64
    (test_spmv.py:105-111); 16-bit only through DeviceMatrix.astype."""
    a = dg.to_dacsr(laplacian_2d(8), 16)
    with pytest.raises(UnsupportedScalarWidth):
        dg.spmv(a, np.ones(a.ncols, np.float16), np.ones(a.nrows, np.float16))
    dm = DeviceMatrix.from_host(a, cuda).astype("float16")
    with pytest.raises(UnsupportedScalarWidth):
        dg.spmv(dm, torch.ones(a.ncols, dtype=torch.float32, device=cuda))


def test_half_c2_full_size_bit_exact(cuda):
    """C2 (128^3 7-pt) with bf16 and f16 values: full-size parity + traffic."""
    csr = laplacian_3d(128)
    a = dg.to_dacsr(csr, 16)
    base = DeviceMatrix.from_host(a, cuda)
    for dtype in ("bfloat16", "float16"):
        dm = base.astype(dtype)
        x = torch.rand(a.ncols, dtype=torch.float64, device=cuda).to(DTYPES[dtype])
        y = dg.spmv(dm, x, None)
        ref = oracle_y("da", dm, x, torch.zeros(a.nrows, dtype=DTYPES[dtype]), 1.0, 0.0, "naive")
        assert np.array_equal(host_bits(y), ref), dtype
