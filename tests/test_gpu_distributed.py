"""Device side of the multi-GPU path on one GPU: the rank-local x_offset /
row-range kernels, the deterministic norm, and the power iteration, all
bit-exact against the CPU oracle.  (NCCL ranks cannot share one GPU; the
exchange logic itself is covered by tests/test_distributed.py on gloo.)"""

import numpy as np
import pytest
import torch

import oracle
from paper_2307_06305_b200 import distributed as D
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.gen import banded_arrays, normal_vector
from paper_2307_06305_b200.power import chunk_partials, fold_ordered, power_iteration
from paper_2307_06305_b200.workloads import BANDED_CONFIGS, normal_table, poisson_cdf

pytestmark = pytest.mark.gpu

N, B, LAM, KMAX, SEED = 1 << 16, 3000, 8.0, 32, 5


def test_sumsq_matches_oracle_restatement(cuda):
    y = normal_vector(300_001, 3, cuda)
    p = chunk_partials(y, 4096)
    want = oracle.sumsq_chunks(y.cpu().numpy(), 4096)
    assert np.array_equal(p.cpu().numpy().view(np.uint64), want.view(np.uint64))
    assert float(fold_ordered(p).item()) == oracle.fold_ordered(want)


@pytest.mark.parametrize("variant", ["naive", "sliced", "sliced_pipe", "tiled"])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_rank_local_blocks_bit_exact(cuda, world, variant):
    arr = banded_arrays(N, B, LAM, KMAX, SEED, cuda, kinds=("da", "csr"))
    full = DeviceMatrix("da", N, N, arr["rowptr"], arr["offsets"], arr["values"])
    x = normal_vector(N, 9, cuda)
    y_full = torch.empty(N, dtype=torch.float64, device=cuda)
    full.spmv_into(x, y_full, 0.75, 0.0, "wstream")
    part = D.RowPartition.equal(N, world, align=1024)
    ys = []
    for rank in range(world):
        plan = D.halo_plan(part, rank, B)
        r0, r1 = part.bounds[rank]
        loc = banded_arrays(N, B, LAM, KMAX, SEED, cuda, r0=r0, r1=r1, kinds=("da", "csr"))
        x_ext = x[plan.lo:plan.hi].clone()        # what the halo exchange delivers
        for kind, inner in (("da", "offsets"), ("csr", "colids")):
            op = D.CudaLocalOp(kind, loc["rowptr"], loc[inner], loc["values"], N, plan, 1024, B,
                               variant=variant)
            y = torch.empty(r1 - r0, dtype=torch.float64, device=cuda)
            for which in range(3):
                op.spmv_part(which, x_ext, y, 0.75)
            if kind == "da":
                ys.append(y)
            else:
                assert torch.equal(y, ys[-1])
    assert torch.equal(torch.cat(ys), y_full)


def test_power_iteration_matches_oracle(cuda):
    arr = banded_arrays(N, B, LAM, KMAX, SEED, cuda)
    dm = DeviceMatrix("da", N, N, arr["rowptr"], arr["offsets"], arr["values"])
    x0 = normal_vector(N, 11, cuda)
    x, norms = power_iteration(dm, x0, iters=8, chunk=4096)
    rp, offs, vals = oracle.gen_fill(N, B, KMAX, SEED, poisson_cdf(LAM, KMAX), normal_table())
    xr = x0.cpu().numpy()
    s = np.sqrt(oracle.fold_ordered(oracle.sumsq_chunks(xr, 4096)))
    for k in range(8):
        xr = oracle.spmv("da", rp, offs, vals, xr, alpha=1.0 / s)
        s = np.sqrt(oracle.fold_ordered(oracle.sumsq_chunks(xr, 4096)))
        assert s == norms[k], k
    assert np.array_equal(x.cpu().numpy().view(np.uint64), (xr * (1.0 / s)).view(np.uint64))


def test_c5_full_size_row_blocks(cuda):
    """Config C5 on one GPU (2^28 rows, ~2.1e9 entries) with the default
    kernel: four contiguous 2^20-row blocks of y (first, last, two interior)
    bit-exact against the oracle on the same rows (host generator)."""
    import os
    n, b, lam, kmax, seed = BANDED_CONFIGS["c5"]
    arr = banded_arrays(n, b, lam, kmax, seed, cuda, kinds=("da",))
    # nnz = 2,147,462,688 for this seed: just under 2^31, so rowptr stays int32
    assert arr["nnz"] > 2_000_000_000
    assert arr["rowptr"].dtype == (torch.int64 if arr["nnz"] > 2**31 - 1 else torch.int32)
    dm = DeviceMatrix("da", n, n, arr["rowptr"], arr["offsets"], arr["values"])
    from paper_2307_06305_b200.spmv import kernel_for
    kernel = kernel_for(dm, "exact", 0)
    assert kernel == "tiled"
    x = normal_vector(n, 21, cuda)
    y = torch.empty(n, dtype=torch.float64, device=cuda)
    dm.spmv_into(x, y, 1.0, 0.0, kernel, 0)
    del arr, dm
    cdf, table = poisson_cdf(lam, kmax), normal_table()
    threads = len(os.sched_getaffinity(0))
    blk = 1 << 20
    for r0 in (0, n // 3 // blk * blk, 2 * n // 3 // blk * blk + 12345, n - blk):
        r1 = r0 + blk
        rp, offs, vals = oracle.gen_fill_parallel(n, b, kmax, seed, cdf, table, r0, r1, threads)
        lo, hi = max(0, r0 - b), min(n, r1 + b)
        xw = oracle.gen_normal(21, lo, hi, table)
        ref = oracle.spmv_kernel("da", rp, offs, vals, xw, np.empty(blk), 1.0, 0.0,
                                 x_offset=r0 - lo)
        got = y[r0:r1].cpu().numpy()
        assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), r0


def test_power_iteration_50_c5_shaped(cuda):
    """50 normalised power iterations on a C5-shaped band (n = 2^22, b =
    32767, Poisson(8)) with the default kernel: every norm and the final
    iterate bit-exact against the oracle's power iteration."""
    import os
    n, b, lam, kmax, seed = 1 << 22, 32767, 8.0, 32, 2027
    arr = banded_arrays(n, b, lam, kmax, seed, cuda, kinds=("da",))
    dm = DeviceMatrix("da", n, n, arr["rowptr"], arr["offsets"], arr["values"])
    x0 = normal_vector(n, 11, cuda)
    x, norms = power_iteration(dm, x0, iters=50, variant="naive")
    threads = len(os.sched_getaffinity(0))
    rp, offs, vals = oracle.gen_fill_parallel(n, b, kmax, seed, poisson_cdf(lam, kmax),
                                              normal_table(), threads=threads)
    xr = x0.cpu().numpy()
    s = np.sqrt(oracle.fold_ordered(oracle.sumsq_chunks(xr, 1 << 16)))
    for k in range(50):
        xr = oracle.spmv("da", rp, offs, vals, xr, alpha=1.0 / s, threads=threads)
        s = np.sqrt(oracle.fold_ordered(oracle.sumsq_chunks(xr, 1 << 16)))
        assert s == norms[k], k
    assert np.array_equal(x.cpu().numpy().view(np.uint64), (xr * (1.0 / s)).view(np.uint64))


def test_nnz_above_2_31_int64_rowptr(cuda):
    """Maximum-size edge: a C5-shaped matrix with nnz > 2^31 (Poisson(8.05)),
    so rowptr must be int64 on the device; sampled rows vs the oracle."""
    n, b, lam, kmax, seed = 1 << 28, 32767, 8.05, 32, 77
    arr = banded_arrays(n, b, lam, kmax, seed, cuda, kinds=("da",))
    assert arr["nnz"] > 2**31 and arr["rowptr"].dtype == torch.int64
    dm = DeviceMatrix("da", n, n, arr["rowptr"], arr["offsets"], arr["values"])
    x = normal_vector(n, 5, cuda)
    cdf, table = poisson_cdf(lam, kmax), normal_table()
    rng = np.random.default_rng(2)
    rows = np.concatenate([[0, n - 1, n // 2], rng.integers(n - (1 << 20), n, 40),
                           rng.integers(0, n, 40)])
    for kernel in ("tiled", "rowblock", "sliced"):
        y = torch.empty(n, dtype=torch.float64, device=cuda)
        dm.spmv_into(x, y, 1.0, 0.0, kernel, 0)
        for r in rows.tolist():
            offs = oracle.gen_row(n, b, kmax, seed, cdf, r)
            acc = 0.0
            for o in offs.tolist():
                xv = oracle.gen_normal(5, r + o, r + o + 1, table)[0]
                acc = acc + oracle.gen_value(b, seed, r, o, table) * xv
            assert acc == float(y[r].item()), (kernel, r)
        del y


@pytest.mark.parametrize("kernel", ["tiled", "sliced_pipe", "wstream", "scalar", "rowblock"])
def test_device_alpha_matches_host_alpha(cuda, kernel):
    """dacsr_spmv_dev_alpha reads alpha from device memory: the same bits as
    passing it by value (the power iteration's 1/s never leaves the GPU)."""
    arr = banded_arrays(N, B, LAM, KMAX, SEED, cuda)
    dm = DeviceMatrix("da", N, N, arr["rowptr"], arr["offsets"], arr["values"])
    x = normal_vector(N, 9, cuda)
    a = 1.0 / 3.7
    y1 = torch.empty(N, dtype=torch.float64, device=cuda)
    y2 = torch.full((N,), 2.0, dtype=torch.float64, device=cuda)
    dm.spmv_into(x, y1, a, 0.0, kernel, 0)
    dm.spmv_into(x, y2, torch.tensor([a], dtype=torch.float64, device=cuda), 0.0, kernel, 0)
    assert torch.equal(y1.view(torch.int64), y2.view(torch.int64))


def test_power_iteration_graph_replay_matches_eager(cuda):
    from paper_2307_06305_b200.power import PowerIteration
    arr = banded_arrays(N, B, LAM, KMAX, SEED, cuda)
    dm = DeviceMatrix("da", N, N, arr["rowptr"], arr["offsets"], arr["values"])
    x0 = normal_vector(N, 11, cuda)
    x_e, n_e = power_iteration(dm, x0, iters=8, chunk=4096)
    pi = PowerIteration(dm, x0, iters=8, chunk=4096, graph=True)
    for _ in range(2):  # replays are repeatable
        pi.run()
        x_g, n_g = pi.result()
        assert n_g == n_e
        assert torch.equal(x_g.view(torch.int64), x_e.view(torch.int64))


def test_fused_norm_in_the_power_iteration(cuda):
    """On the TILED kernel the power iteration takes ||y||^2 from the SpMV's
    epilogue (512-row group sums); the norms and the iterate equal the
    separate-pass run's, and the three-launch rank-local operator returns the
    same chunk partials."""
    from paper_2307_06305_b200.power import PowerIteration
    n, b = 1 << 17, 20000
    arr = banded_arrays(n, b, 5.0, 12, SEED, cuda)  # <= 12 entries per row: none left out
    dm = DeviceMatrix("da", n, n, arr["rowptr"], arr["offsets"], arr["values"])
    x0 = normal_vector(n, 11, cuda)
    fused = PowerIteration(dm, x0, iters=6, chunk=4096, variant="tiled")
    assert fused.fused
    fused.run()
    xf, nf = fused.result()
    plain = PowerIteration(dm, x0, iters=6, chunk=4096, variant="tiled")
    plain.fused, plain.group_sumsq = False, None
    plain.run()
    xp, npl = plain.result()
    assert nf == npl and torch.equal(xf.view(torch.int64), xp.view(torch.int64))
    # one rank's operator: interior + two strips, cuts on group boundaries
    part = D.RowPartition.equal(n, 1, align=4096)
    plan = D.halo_plan(part, 0, b)
    op = D.CudaLocalOp("da", arr["rowptr"], arr["offsets"], arr["values"], n, plan, 4096, b)
    assert op.fused and all(r0 % 512 == 0 and r1 % 512 == 0 for r0, r1 in op.ranges)
    alpha = torch.tensor([0.5], dtype=torch.float64, device=cuda)
    x_ext = x0[plan.lo:plan.hi].clone()
    y = torch.empty(n, dtype=torch.float64, device=cuda)
    for which in range(3):
        op.spmv_part(which, x_ext, y, alpha)
    got = op.partials_after_spmv(y).cpu().numpy()
    want = op.partials(y).cpu().numpy()
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
