"""The band-tiled device layout (dacsr_tiles_t) and the TILED kernel — needs a B200.

The layout is a bit-for-bit re-arrangement of the CSR/DA-CSR entries (512-row
groups, column tiles, pair-step packed lane lists); the kernel folds every
row from +0.0 in column order, i.e. the reference's naive order
(_numba_kernels.py:82-91), so every result here is BIT-EXACT against the
reference outputs (tests/golden) and the oracle.  Rows with more than 15
entries inside one tile are left out of the layout and reduced warp by warp;
small tile widths force that path, many tiles per group and partial tiles.
"""

import numpy as np
import pytest
import torch

import oracle
import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.gen import banded_arrays, normal_vector
from paper_2307_06305_b200.workloads import add_skew_rows, laplacian_2d, uniform_x
from test_gpu_parity import bits, host_matrix
from test_oracle import CORPUS

pytestmark = pytest.mark.gpu


def untile(dm):
    """Decode the layout: {row: [(tile, inner, value), ...]} in storage order,
    the skip masks and the left-out row list."""
    _, tl, t = dm._tiled
    ptrs = t["ptrs"].cpu().numpy()
    cnt_ptr, ent_ptr = ptrs[0], ptrs[1]
    tile_lo = t["tile_lo"].cpu().numpy()
    counts = t["counts"].cpu().numpy().view(np.uint64)
    order = t["order"].cpu().numpy().view(np.uint64)
    masks = t["masks"].cpu().numpy().view(np.uint64)
    inner, vals = t["inner"].cpu().numpy(), t["values"].cpu().numpy()
    rows = {}
    for g in range(tl.ngroups):
        pos = int(ent_ptr[g])
        for k in range(int(cnt_ptr[g + 1] - cnt_ptr[g])):
            b = int(cnt_ptr[g]) + k
            cw = [int(w) for w in counts[b * 32:(b + 1) * 32]]
            ow = [int(w) for w in order[b * 32:(b + 1) * 32]]
            mw = int(masks[b])
            # lane l: its rows in fold order (k-th: slot j = nibble k of ow,
            # n = nibble k of cw; the list ends at the first n = 0)
            seq = []
            for l in range(32):
                s_l = []
                for q in range(16):
                    n = (cw[l] >> (4 * q)) & 15
                    if n == 0:
                        assert cw[l] >> (4 * q) == 0
                        break
                    s_l.append(((ow[l] >> (4 * q)) & 15, n))
                js = [j for j, _ in s_l]
                assert len(set(js)) == len(js)
                seq.append(s_l)
            tot = [sum(n for _, n in s_l) for s_l in seq]
            lists = [[] for _ in range(32)]
            G = tl.step_group
            for q in range((max(tot) + G - 1) // G):
                for l in range(32):
                    if G * q < tot[l]:
                        lists[l] += list(range(pos, pos + G))
                        pos += G
            for l in range(32):
                slots = iter(lists[l])
                for j, n in seq[l]:
                    r = tl.row_start + 512 * g + 32 * j + (l ^ ((mw >> (4 * j)) & 15))
                    for _ in range(n):
                        p = next(slots)
                        rows.setdefault(r, []).append((int(tile_lo[g]) + k, inner[p], vals[p]))
        assert pos == ent_ptr[g + 1]
    skip = t["skip"].cpu().numpy().view(np.uint16)
    return rows, skip, t["ovf_rows"].cpu().numpy()[:tl.n_ovf]


@pytest.mark.parametrize("kind", ["csr", "da"])
def test_layout_is_a_rearrangement(cuda, kind):
    for c in CORPUS[::5]:
        a = host_matrix(c, kind)
        dm = DeviceMatrix.from_host(a, cuda)
        rp = np.asarray(a.rowptr, dtype=np.int64)
        for tc in (64, 128, 8192):
            dm.build_tiles(tc)
            tl = dm._tiled[1]
            rows, skip, ovf = untile(dm)
            assert list(ovf) == sorted(ovf)
            assert not set(rows) & set(int(r) for r in ovf)
            for r in range(a.nrows):
                b, e = rp[r], rp[r + 1]
                if r in set(int(v) for v in ovf):
                    continue
                got = rows.get(r, [])
                assert len(got) == e - b, (r, tc)
                cols = np.asarray(a.colids)[b:e].astype(np.int64) + (r if kind == "da" else 0)
                for i, (tile, inn, val) in enumerate(got):
                    assert inn == np.asarray(a.colids)[b + i]
                    assert bits(np.array([val])) .tobytes() == bits(np.asarray(a.values)[b + i:b + i + 1]).tobytes()
                    assert tile == (cols[i] - tl.col0) // tc


@pytest.mark.parametrize("kind", ["csr", "da"])
@pytest.mark.parametrize("tile_cols", [None, 64, 256])
def test_golden_bit_exact(cuda, kind, tile_cols):
    for k, c in enumerate(CORPUS):
        dm = DeviceMatrix.from_host(host_matrix(c, kind), cuda)
        dm.build_tiles(tile_cols)
        x = torch.from_numpy(c["x"]).to(cuda)
        y = torch.from_numpy(c["y0"].copy()).to(cuda)
        out = dg.spmv(dm, x, y, c["alpha"], c["beta"], "tiled")
        assert out is y
        assert np.array_equal(bits(y.cpu().numpy()), bits(c["y_naive"])), (k, kind, tile_cols)


@pytest.mark.parametrize("kind", ["csr", "da"])
def test_wide_band_left_out_rows_ranges_x_offset(cuda, kind):
    """Random band (C3 shape, small n): tiny tiles leave rows out; every row
    range and a rank-local halo buffer (x_offset) stay bit-exact."""
    n, b = 1 << 14, 3000
    arr = banded_arrays(n, b, 16.0, 64, 5, cuda, kinds=("da", "csr"))
    rp = arr["rowptr"].cpu().numpy()
    offs = arr["offsets"].cpu().numpy()
    vals = arr["values"].cpu().numpy()
    dm = DeviceMatrix(kind, n, n, arr["rowptr"], arr["offsets" if kind == "da" else "colids"],
                      arr["values"])
    xh = normal_vector(n, 3, cuda).cpu().numpy()
    pad = 41
    x_ext = torch.zeros(n + 2 * pad, dtype=torch.float64, device=cuda)
    x_ext[pad:pad + n] = torch.from_numpy(xh).to(cuda)
    rng = np.random.default_rng(4)
    for tc in (4096, 6000 // 16 * 16):
        dm.build_tiles(tc)
        assert dm.tiles_info()["n_ovf"] > 0
        for _ in range(6):
            r0, r1 = sorted(int(v) for v in rng.integers(0, n + 1, 2))
            y0 = rng.uniform(-1, 1, n)
            y = torch.from_numpy(y0.copy()).to(cuda)
            dm.spmv_into(x_ext, y, 0.7, -0.3, "tiled", 0, x_offset=pad, row_start=r0, row_end=r1)
            ref = oracle.spmv_kernel("da", rp, offs, vals, xh, y0.copy(), 0.7, -0.3,
                                     row_start=r0, row_end=r1)
            assert np.array_equal(bits(y.cpu().numpy()), bits(ref)), (tc, r0, r1)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16])
def test_narrow_values_match_exact_kernels(cuda, dtype):
    n = 1 << 15
    arr = banded_arrays(n, 32767, 8.0, 32, 6, cuda, kinds=("da",))
    dm = DeviceMatrix("da", n, n, arr["rowptr"], arr["offsets"], arr["values"]).astype(dtype)
    x = normal_vector(n, 9, cuda).to(dtype)
    want = dm.spmv_into(x, torch.empty(n, dtype=dtype, device=cuda), 1.0, 0.0, "scalar")
    got = dm.spmv_into(x, torch.empty(n, dtype=dtype, device=cuda), 1.0, 0.0, "tiled")
    as_int = {4: torch.int32, 2: torch.int16}[dtype.itemsize]
    assert torch.equal(got.view(as_int), want.view(as_int))
    from paper_2307_06305_b200 import _native
    assert dm.tiles_info()["tile_cols"] == _native.lib().dacsr_tiles_max_cols(dm.desc.values_dtype)


def test_skewed_rows_and_default_selection(cuda):
    """Skewed stencil (C4-like): the tiled kernel stays exact with long rows
    left out; the default selection keeps SLICED_PIPE for it."""
    a = dg.to_dacsr(add_skew_rows(laplacian_2d(256), frac=0.02, alpha=0.5, cap=1200, band=700,
                                  seed=3), 16)
    dm = DeviceMatrix.from_host(a, cuda)
    x = torch.from_numpy(uniform_x(a.ncols, 5)).to(cuda)
    ref = oracle.spmv("da", a.rowptr, a.colids, a.values, x.cpu().numpy())
    for tc in (64, 1024, 8192):
        dm.build_tiles(tc)
        y = dg.spmv(dm, x, variant="tiled")
        assert np.array_equal(bits(y.cpu().numpy()), bits(ref)), tc
    assert dm.stats.scatter < 0.5
    from paper_2307_06305_b200.spmv import kernel_for
    assert kernel_for(dm, "exact", 0) == "sliced_pipe"


def test_fused_group_sumsq(cuda):
    """spmv_into(group_sumsq=...) stores the sums of y^2 of whole 512-row
    groups in the fixed group tree: the chunk partials folded from them are
    the bits dacsr_sumsq_chunks computes from y (and the oracle restates);
    row ranges made of whole groups write only their groups; anything else
    is refused."""
    from paper_2307_06305_b200.errors import DeviceError
    from paper_2307_06305_b200.power import chunk_partials, partials_from_groups
    n = (1 << 15) + 777  # the last group is partial
    arr = banded_arrays(n, 2000, 5.0, 12, 6, cuda, kinds=("da",))  # <= 12 entries per row
    dm = DeviceMatrix("da", n, n, arr["rowptr"], arr["offsets"], arr["values"])
    dm.build_tiles()
    assert dm.tiles_info()["n_ovf"] == 0 and dm.fused_sumsq_ok("tiled")
    x = normal_vector(n, 9, cuda)
    alpha = torch.tensor([0.37], dtype=torch.float64, device=cuda)
    ng = (n + 511) // 512
    gs = torch.full((ng,), float("nan"), dtype=torch.float64, device=cuda)
    y = torch.empty(n, dtype=torch.float64, device=cuda)
    dm.spmv_into(x, y, alpha, 0.0, "tiled", 0, group_sumsq=gs)
    y2 = dm.spmv_into(x, torch.empty_like(y), alpha, 0.0, "tiled", 0)
    assert torch.equal(y.view(torch.int64), y2.view(torch.int64))
    for chunk in (512, 4096, 1 << 16):
        fused = partials_from_groups(gs, n, chunk).cpu().numpy()
        direct = chunk_partials(y, chunk).cpu().numpy()
        assert np.array_equal(fused.view(np.uint64), direct.view(np.uint64)), chunk
        want = oracle.sumsq_chunks(y.cpu().numpy(), chunk)
        assert np.array_equal(fused.view(np.uint64), want.view(np.uint64)), chunk
    # beta != 0 and a range of whole groups: only its groups are written
    gs2 = torch.full((ng,), -1.0, dtype=torch.float64, device=cuda)
    y3 = y.clone()
    dm.spmv_into(x, y3, alpha, 0.5, "tiled", 0, row_start=1024, row_end=8192, group_sumsq=gs2)
    g2 = gs2.cpu().numpy()
    assert (g2[:2] == -1.0).all() and (g2[16:] == -1.0).all()
    want = oracle.sumsq_chunks(y3.cpu().numpy()[1024:8192], 512)
    assert np.array_equal(g2[2:16].view(np.uint64), want.view(np.uint64))
    assert dm.fused_sumsq_ok("tiled", 0, 1024, 8192)
    # ranges that cut a group, other kernels
    assert not dm.fused_sumsq_ok("tiled", 0, 100, 8192)
    with pytest.raises(DeviceError):
        dm.spmv_into(x, y3, alpha, 0.0, "tiled", 0, row_start=100, row_end=8192, group_sumsq=gs2)
    assert not dm.fused_sumsq_ok("sliced_pipe")
    with pytest.raises(DeviceError):
        dm.spmv_into(x, y3, alpha, 0.0, "sliced_pipe", 0, group_sumsq=gs2)


def test_selection_falls_back_when_rows_do_not_fit_the_tiles(cuda):
    """Dense rows in a narrow random band: the gathers are scattered (the
    statistic says TILED) but most rows hold more than 15 entries inside one
    column tile and would be left to the warp-per-row pass — the default
    selection builds the layout, sees that, and runs SLICED_PIPE instead."""
    from paper_2307_06305_b200.spmv import kernel_for
    n = 1 << 15
    arr = banded_arrays(n, 1000, 40.0, 64, 8, cuda, kinds=("da",))
    dm = DeviceMatrix("da", n, n, arr["rowptr"], arr["offsets"], arr["values"])
    assert dm.stats.scatter > 0.5
    assert kernel_for(dm, "exact", 0) == "sliced_pipe" and dm._tiled is None
    x = normal_vector(n, 4, cuda)
    y = dg.spmv(dm, x)
    ref = oracle.spmv("da", arr["rowptr"].cpu().numpy(), arr["offsets"].cpu().numpy(),
                      arr["values"].cpu().numpy(), x.cpu().numpy())
    assert np.array_equal(bits(y.cpu().numpy()), bits(ref))
    # the explicit variant still runs the tiled kernel (left-out rows and all)
    y2 = dg.spmv(dm, x, variant="tiled")
    assert dm.tiles_info()["n_ovf"] > n // 2
    assert np.array_equal(bits(y2.cpu().numpy()), bits(ref))
