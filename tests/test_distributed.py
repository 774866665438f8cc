"""Multi-rank row-block SpMV / power iteration on CPU with gloo (world 2).

The local multiply is the CPU oracle (test infrastructure) behind the same
LocalOp interface the CUDA path implements; what is tested here is the
host logic: partition, halo plans, the P2P exchange, the x_offset
addressing, the rank-ordered deterministic norm — and that 1 and 2 ranks
give bit-identical iterates.
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2307_06305_b200 import distributed as D
from paper_2307_06305_b200.workloads import normal_table, poisson_cdf

N, B, LAM, KMAX, SEED = 1 << 13, 300, 8.0, 32, 7
CHUNK = 512
ITERS = 6


def test_partition_and_halo_plans():
    part = D.RowPartition.equal(1000, 4, align=64)
    assert part.bounds[0][0] == 0 and part.bounds[-1][1] == 1000
    assert all(a % 64 == 0 for a, _ in part.bounds)
    p1 = D.halo_plan(part, 1, 50)
    r0, r1 = part.bounds[1]
    assert p1.lo == r0 - 50 and p1.hi == r1 + 50 and p1.x_offset == 50
    assert {q for q, *_ in p1.recv} == {0, 2} and {q for q, *_ in p1.send} == {0, 2}
    # wide halo spanning several owners
    part = D.RowPartition.equal(100, 5)
    p2 = D.halo_plan(part, 2, 45)
    got = sorted((q, g0, g1) for q, g0, g1 in p2.recv)
    assert got == [(0, 0, 20), (1, 20, 40), (3, 60, 80), (4, 80, 100)]
    # every recv has a matching send on the owner
    for rank in range(5):
        for q, g0, g1 in D.halo_plan(part, rank, 45).recv:
            assert (rank, g0, g1) in {(t, a, b) for t, a, b in D.halo_plan(part, q, 45).send}
    rp = np.concatenate([[0], np.cumsum(np.r_[np.full(50, 10), np.full(50, 1)])])
    bal = D.RowPartition.nnz_balanced(rp, 2, align=5)
    assert bal.bounds[0][1] % 5 == 0 and 20 <= bal.bounds[0][1] <= 30


class OracleLocalOp:
    """CPU stand-in for CudaLocalOp (oracle kernels; test-only)."""

    def __init__(self, rowptr, offsets, values, plan):
        self.rowptr, self.offsets, self.values, self.plan = rowptr, offsets, values, plan

    def spmv_part(self, which, x_ext, y, alpha, stream=None):
        if which == 0:
            oracle.spmv_kernel("da", self.rowptr, self.offsets, self.values, x_ext.numpy(),
                               y.numpy(), alpha, 0.0, x_offset=self.plan.x_offset)

    def partials(self, y):
        return torch.from_numpy(oracle.sumsq_chunks(y.numpy(), CHUNK))

    def fold(self, allp):
        return oracle.fold_ordered(allp.numpy())


def _local_problem(rank, world):
    part = D.RowPartition.equal(N, world, align=CHUNK)
    plan = D.halo_plan(part, rank, B)
    r0, r1 = part.bounds[rank]
    rp, offs, vals = oracle.gen_fill(N, B, KMAX, SEED, poisson_cdf(LAM, KMAX), normal_table(),
                                     r0, r1)
    x0 = oracle.gen_normal(11, r0, r1, normal_table())
    return plan, OracleLocalOp(rp, offs, vals, plan), torch.from_numpy(x0)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan, op, x0 = _local_problem(rank, world)
        part = D.RowPartition.equal(N, world, align=CHUNK)
        # world 1 exchanges the counts, world 2 uses the partition's (both paths)
        counts = D.chunk_counts(part, CHUNK) if world > 1 else None
        x, norms = D.power_iteration(op, plan, x0, ITERS, overlap=False, counts=counts)
        np.save(f"{out}/x{rank}.npy", x.numpy())
        np.save(f"{out}/norms{rank}.npy", np.array(norms))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world):
    out = tempfile.mkdtemp()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="fork")
    x = np.concatenate([np.load(f"{out}/x{r}.npy") for r in range(world)])
    norms = [np.load(f"{out}/norms{r}.npy") for r in range(world)]
    return x, norms


def _reference_power_iteration():
    """Single-process CPU power iteration with the reference API's alpha."""
    rp, offs, vals = oracle.gen_fill(N, B, KMAX, SEED, poisson_cdf(LAM, KMAX), normal_table())
    x = oracle.gen_normal(11, 0, N, normal_table())
    s = np.sqrt(oracle.fold_ordered(oracle.sumsq_chunks(x, CHUNK)))
    norms = []
    for _ in range(ITERS):
        y = oracle.spmv("da", rp, offs, vals, x, alpha=1.0 / s)
        s = np.sqrt(oracle.fold_ordered(oracle.sumsq_chunks(y, CHUNK)))
        norms.append(s)
        x = y
    return x * (1.0 / s), norms


@pytest.mark.timeout(300)
def test_gloo_two_ranks_bit_identical_to_one():
    x1, n1 = _run(1)
    x2, n2 = _run(2)
    assert np.array_equal(x1.view(np.uint64), x2.view(np.uint64))
    assert np.array_equal(n1[0], n2[0]) and np.array_equal(n2[0], n2[1])
    xr, nr = _reference_power_iteration()
    assert np.array_equal(np.array(nr), n1[0])
    assert np.array_equal(xr.view(np.uint64), x1.view(np.uint64))


def test_launch_ranges_cover_rows_on_group_boundaries():
    """A rank's interior / strip launches: disjoint, covering, the interior
    free of halo rows, every cut a multiple of 512 (fused group sums)."""
    for n_local in (0, 100, 512, 65536, 1 << 20, (1 << 20) + 65536):
        for b in (1, 511, 512, 3000, 32767, 1 << 21):
            (i0, i1), (a0, a1), (c0, c1) = D.launch_ranges(n_local, b)
            assert a0 == 0 and a1 == i0 and i1 == c0 and c1 == n_local and i0 <= i1
            assert i0 % 512 == 0 or i0 == n_local
            assert i1 % 512 == 0 or i1 == i0
            if i1 > i0:  # interior rows read no halo
                assert i0 >= b and i1 <= n_local - b
            # the strips are as thin as the group grid allows
            assert i0 <= min(n_local, b + 511) and (i1 == i0 or i1 > n_local - b - 512)
