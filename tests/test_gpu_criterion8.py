"""Reference acceptance criterion 8 restated for the GPU — needs a B200.

The reference (pkg/tests/test_acceptance.py:315-375) times the best variant
of each format on matrices whose traffic is far beyond the last-level cache
and requires best DA-CSR(i16) to beat best CSR(i32) — gated on a measured
precondition: the best CSR run must stream at >= 0.6x the machine's copy
bandwidth (otherwise the kernel is not memory-bound and byte savings cannot
surface).  Here: configs C2, C3 and C4 (BASELINE.json) and C2's stencil at
8 times its rows (1.5 GB), each SpMV timed cold
(L2 flushed before it, so the operator streams from HBM), the fastest exact
kernel per format (DeviceMatrix.autotune, cold), and the copy bandwidth
measured on this device the reference's way (best of 5 copies of a 200 MB
array, read + write bytes).
"""

import numpy as np
import pytest
import torch

import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.harness import time_kernel
from paper_2307_06305_b200.model import StorageWidths, spmv_traffic

pytestmark = pytest.mark.gpu


def copy_gbs(device):
    src = torch.rand(25_000_000, dtype=torch.float64, device=device)
    dst = torch.empty_like(src)
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dst.copy_(src)
        e1.record()
        e1.synchronize()
        best = max(best, 2 * src.numel() * 8 / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return best


def best_cold(dm, x):
    dm.autotune(cold=True, x=x, reps=3)
    y = torch.empty(dm.nrows, dtype=dm.values.dtype, device=dm.device)
    k = dm.tuned_kernel
    fn = lambda: dm.spmv_into(x, y, 1.0, 0.0, k, 0)
    return time_kernel(fn, epochs=3, warmup_iters=1, min_epoch_iters=3, min_epoch_time=0.0,
                       cold=True), k


def pair(config, device):
    if config == "c3":
        from paper_2307_06305_b200.gen import banded_device, normal_vector
        mats = banded_device("c3", device)
        return mats["csr"], mats["da"], normal_vector(mats["da"].ncols, 17, device)
    from paper_2307_06305_b200.workloads import (laplacian_3d, laplacian_3d_box,
                                                 skewed_rcm_laplacian, uniform_x)
    a = (laplacian_3d(128) if config == "c2" else
         laplacian_3d_box((1024, 128, 128)) if config == "c2xl" else skewed_rcm_laplacian(2048)[0])
    x = torch.from_numpy(uniform_x(a.ncols, 1)).to(device)
    return DeviceMatrix.from_host(a, device), DeviceMatrix.from_host(dg.to_dacsr(a, 16), device), x


@pytest.mark.parametrize("config", [
    "c2",
    # C2's stencil on a 1024 x 128 x 128 box (1.5 GB, int16 offsets): the
    # stencil class far out of L2, as the reference's criterion asks —
    # measured DA/CSR 1.10-1.12 cold, 1.08 in back-to-back SpMVs
    "c2xl",
    # C4: DA/CSR 1.09-1.11 cold since the long rows' fold stopped setting the
    # kernel's time (it measured 0.996 .. 1.063 before, an expected failure
    # then; profiles/r2_sliced_c4_ab.txt)
    "c4",
    # TILED (the C3 kernel): measured DA/CSR 1.13 cold
    "c3",
])
def test_criterion_8_measured_speedup_direction(cuda, config):
    csr, da, x = pair(config, cuda)
    t_csr, k_csr = best_cold(csr, x)
    t_da, k_da = best_cold(da, x)
    bytes_csr = spmv_traffic(csr.nrows, csr.ncols, csr.nnz,
                             StorageWidths(csr.oindex_width // 8, 4, 8)).total_bytes
    spmv = bytes_csr / t_csr / 1e9
    cp = copy_gbs(cuda)
    ratio = t_csr / t_da
    detail = (f"{config}: best dacsr(i16) [{k_da}] vs csr(i32) [{k_csr}] {ratio:.3f}x cold; "
              f"csr {spmv:.0f} GB/s vs copy {cp:.0f} GB/s")
    print(f"\n[criterion 8] {detail}")
    if spmv < 0.6 * cp:
        pytest.skip(f"not memory-bound here (precondition of the reference criterion): {detail}")
    assert ratio > 1.0, detail
