"""BASELINE configs at full size on the GPU: generator parity, size-
independent properties, and sampled-row parity against the oracle."""

import numpy as np
import pytest
import torch

import oracle
import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.gen import banded_arrays, banded_device, normal_vector
from paper_2307_06305_b200.workloads import BANDED_CONFIGS, normal_table, poisson_cdf

pytestmark = pytest.mark.gpu


def test_generator_bit_exact_small(cuda):
    n, b, lam, kmax, seed = 1 << 15, 3000, 16.0, 64, 99
    arr = banded_arrays(n, b, lam, kmax, seed, cuda, kinds=("da", "csr"))
    rp, offs, vals = oracle.gen_fill(n, b, kmax, seed, poisson_cdf(lam, kmax), normal_table())
    assert np.array_equal(arr["rowptr"].cpu().numpy().astype(np.int64), rp)
    assert np.array_equal(arr["offsets"].cpu().numpy(), offs)
    assert np.array_equal(arr["values"].cpu().numpy().view(np.uint64), vals.view(np.uint64))
    rows = np.repeat(np.arange(n), np.diff(rp))
    assert np.array_equal(arr["colids"].cpu().numpy(), rows + offs)
    # a row block generated alone equals the same rows of the whole matrix
    part = banded_arrays(n, b, lam, kmax, seed, cuda, r0=1000, r1=5000, kinds=("da",))
    e0, e1 = rp[1000], rp[5000]
    assert np.array_equal(part["offsets"].cpu().numpy(), offs[e0:e1])
    xd = normal_vector(4096, 7, cuda).cpu().numpy()
    assert np.array_equal(xd.view(np.uint64), oracle.gen_normal(7, 0, 4096, normal_table()).view(np.uint64))


def _sample_rows(dm, rows):
    rp = dm.rowptr.cpu().numpy().astype(np.int64)
    out = []
    for r in rows:
        s, e = rp[r], rp[r + 1]
        out.append((dm.colids[s:e].cpu().numpy(), dm.values[s:e].cpu().numpy()))
    return out


def test_c3_full_size(cuda):
    n, b, lam, kmax, seed = BANDED_CONFIGS["c3"]
    mats = banded_device("c3", cuda)
    da, csr = mats["da"], mats["csr"]
    assert da.nnz > 250_000_000 and da.colids.dtype == torch.int16
    assert da.rowptr.dtype == torch.int32
    # sampled rows equal the oracle generator
    rng = np.random.default_rng(0)
    rows = np.concatenate([[0, 1, n - 1, n - 2], rng.integers(0, n, 300)])
    cdf, table = poisson_cdf(lam, kmax), normal_table()
    for r, (offs, vals) in zip(rows, _sample_rows(da, rows)):
        want = oracle.gen_row(n, b, kmax, seed, cdf, int(r))
        assert np.array_equal(offs.astype(np.int32), want)
        assert all(vals[i] == oracle.gen_value(b, seed, int(r), int(o), table)
                   for i, o in enumerate(want))
    x = normal_vector(n, 17, cuda)
    # the row-statistics selection sends this random band to TILED
    from paper_2307_06305_b200.spmv import kernel_for
    assert da.stats.scatter > 0.9 and kernel_for(da, "exact", 0) == "tiled"
    assert kernel_for(csr, "exact", 0) == "tiled"
    yd = dg.spmv(da, x, variant="naive")
    yc = dg.spmv(csr, x, variant="naive")
    assert torch.equal(yd, yc)  # naive CSR == naive DA bit-exact (reference crit 4)
    # the FULL y against the oracle (the reference's naive kernel restated in
    # C, all host threads), DA and CSR
    import os
    rp = da.rowptr.cpu().numpy()
    xh = x.cpu().numpy()
    ref = oracle.spmv("da", rp, da.colids.cpu().numpy(), da.values.cpu().numpy(), xh,
                      threads=len(os.sched_getaffinity(0)))
    assert np.array_equal(yd.cpu().numpy().view(np.uint64), ref.view(np.uint64))
    ref_c = oracle.spmv("csr", rp, csr.colids.cpu().numpy(), csr.values.cpu().numpy(), xh,
                        threads=len(os.sched_getaffinity(0)))
    assert np.array_equal(ref_c.view(np.uint64), ref.view(np.uint64))
    del ref_c
    # every exact kernel (both layouts) gives the same bits at full size
    for dm in (da, csr):
        for kernel in ("sliced", "sliced_pipe", "tiled", "wstream", "scalar"):
            yk = torch.empty(n, dtype=torch.float64, device=cuda)
            dm.spmv_into(x, yk, 1.0, 0.0, kernel, 0)
            assert torch.equal(yk, yd), (dm.kind, kernel)
        dm._sliced = None
        dm._tiled = None
        dm._launch_cache.clear()
    # sampled rows against the oracle kernel on the copied row data
    yh = yd.cpu().numpy()
    for r, (offs, vals) in zip(rows, _sample_rows(da, rows)):
        rp = np.array([0, len(offs)], np.int64)
        yr = np.empty(1)
        # a 1-row DA matrix at global row r: shift x so that row 0 reads x[r + off]
        oracle.spmv_kernel("csr", rp, offs.astype(np.int64) + r, vals, xh, yr, 1.0, 0.0)
        assert yr[0] == yh[r]
    # linearity: A(x1 + x2) ≈ A x1 + A x2 (exact product rounding differs)
    x2 = normal_vector(n, 18, cuda)
    y12 = dg.spmv(da, x + x2, variant="naive")
    y2 = dg.spmv(da, x2, variant="naive")
    err = (y12 - yd - y2).abs().max().item()
    assert err <= 1e-12 * y12.abs().max().item() * 64
    for variant in ("vector4", "vector8", "rowblock_tree", "multi_accumulator_3"):
        yv = dg.spmv(da, x, variant=variant)
        rel = (yv - yd).abs().max().item() / yd.abs().max().item()
        assert rel <= 2.0 ** -40, (variant, rel)


def test_c4_rcm_and_skew(cuda):
    import hashlib
    import json
    import os
    from conftest import GOLDEN
    from paper_2307_06305_b200.workloads import skewed_rcm_laplacian
    with open(os.path.join(GOLDEN, "c4_rcm.json")) as f:
        g = json.load(f)
    a, info = skewed_rcm_laplacian(g["nx"], scramble_seed=g["scramble_seed"])
    perm_hash = hashlib.sha256(np.ascontiguousarray(info["perm"], np.int64).tobytes()).hexdigest()
    assert perm_hash == g["perm_sha256"]          # product RCM == reference rcm()
    assert info["bandwidth_rcm"] == g["bandwidth_rcm"]
    d = dg.to_dacsr(a, 16)
    x = np.random.default_rng(3).uniform(-1, 1, a.ncols)
    for variant in ("naive", "strip_mined_4", "sliced", "sliced_pipe", "tiled"):
        y = dg.spmv(d, x, variant=variant)
        order = variant if variant in ("naive", "strip_mined_4") else "naive"
        ref = oracle.spmv("da", d.rowptr, d.colids, d.values, x, order=order, threads=8)
        assert np.array_equal(y.view(np.uint64), ref.view(np.uint64)), variant


def test_large_regular_operator_default_kernel(cuda):
    """A stencil well out of L2 (4M rows, C2's stencil on a 256 x 128 x 128
    box): the default stays SLICED_PIPE (with 32-bit slice indices it beats
    SLICED and WSTREAM at every size measured, tools/stream_vs_sliced.py) and
    gives the oracle's bits."""
    from paper_2307_06305_b200.device import DeviceMatrix
    from paper_2307_06305_b200.spmv import kernel_for
    from paper_2307_06305_b200.workloads import laplacian_3d_box, uniform_x
    big = dg.to_dacsr(laplacian_3d_box((256, 128, 128)), 16)
    dm = DeviceMatrix.from_host(big, cuda)
    assert dm.stats.rows == 1 << 22 and kernel_for(dm, "exact", 0) == "sliced_pipe"
    x = torch.from_numpy(uniform_x(big.ncols, 3)).to(cuda)
    ref = oracle.spmv("da", big.rowptr, big.colids, big.values, x.cpu().numpy())
    for variant in ("naive", "sliced", "wstream"):
        y = dg.spmv(dm, x, variant=variant)
        assert np.array_equal(y.cpu().numpy().view(np.uint64), ref.view(np.uint64)), variant
