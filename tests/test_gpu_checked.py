"""Bounds-checked build (the compute-sanitizer substitute; sanitizer runs
are closed on this pool): every kernel of libdacsr_b200_checked.so traps on
an entry, row, column or staging-window index out of range.  The golden
corpus and the skewed/empty-chunk cases run through it in a subprocess (a
trap poisons the CUDA context), results still bit-exact."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

DRIVER = r'''
import sys
sys.path[:0] = [".", "tests", "oracle"]
import numpy as np, torch
import oracle
import paper_2307_06305_b200 as dg
from paper_2307_06305_b200 import _native
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.workloads import add_skew_rows, laplacian_2d, uniform_x
from test_oracle import CORPUS
assert _native.LIB_PATH.endswith("_checked.so"), _native.LIB_PATH
dev = torch.device("cuda")
kernels = ("sliced", "sliced_pipe", "tiled", "wstream", "rowblock", "staged", "scalar", "vector4", "warp", "rowblock_tree",
           "multi_accumulator_3", "strip_mined_4")
for c in CORPUS:
    for kind, inner in (("csr", "colids"), ("da", "offsets")):
        cls = dg.CsrMatrix if kind == "csr" else dg.DacsrMatrix
        dm = DeviceMatrix.from_host(cls(c["nrows"], c["ncols"], c["rowptr"], c[inner], c["values"]), dev)
        x = torch.from_numpy(c["x"]).to(dev)
        for v in kernels:
            y = torch.from_numpy(c["y0"].copy()).to(dev)
            dg.spmv(dm, x, y, c["alpha"], c["beta"], v)
a = add_skew_rows(laplacian_2d(128), frac=0.02, alpha=0.1, cap=3000, band=900, seed=2)
d = dg.to_dacsr(a, 16)
dm = DeviceMatrix.from_host(d, dev)
x = torch.from_numpy(uniform_x(a.ncols, 1)).to(dev)
ref = oracle.spmv("da", d.rowptr, d.colids, d.values, x.cpu().numpy())
for rows in (32, 64):
    for vcap in (64, 160, 2048):
        dm.set_chunk_window(vcap, rows)
        y = dg.spmv(dm, x, variant="wstream")
        assert np.array_equal(y.cpu().numpy(), ref)
for max_len, medium_len in ((1, 1), (3, 3), (5, 40), (40, 254)):
    dm.build_slices(max_len, medium_len)
    for v in ("sliced", "sliced_pipe", "tiled"):
        y = dg.spmv(dm, x, variant=v)
        assert np.array_equal(y.cpu().numpy(), ref)
for tc in (64, 256, 4096):  # many tiles, left-out rows, partial last tiles
    dm.build_tiles(tc)
    y = dg.spmv(dm, x, variant="tiled")
    assert np.array_equal(y.cpu().numpy(), ref)
    xe = torch.zeros(a.ncols + 77, dtype=torch.float64, device=dev)
    xe[37:37 + a.ncols] = x
    y = torch.full((a.nrows,), 3.0, dtype=torch.float64, device=dev)
    dm.spmv_into(xe, y, 1.0, 0.0, "tiled", 0, x_offset=37, row_start=700, row_end=9000)
    assert np.array_equal(y.cpu().numpy()[700:9000], ref[700:9000])
for v in kernels:
    y = dg.spmv(dm, x, variant=v)
torch.cuda.synchronize()
print("checked build: clean")
'''


def test_checked_build_runs_clean(cuda):
    lib = os.path.join(ROOT, "paper_2307_06305_b200", "lib", "libdacsr_b200_checked.so")
    if not os.path.exists(lib):
        pytest.skip("checked library not built (build() builds it)")
    env = dict(os.environ, DACSR_LIB="checked")
    r = subprocess.run([sys.executable, "-c", DRIVER], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "checked build: clean" in r.stdout
