"""Row-block multi-GPU SpMV with a ±bandwidth halo of x.

Partition: contiguous row blocks [r0, r1) per rank — equal rows, or nnz-
balanced with the reference's ``row_blocks`` rule (spmv/__init__.py:71-85)
— with every boundary on a multiple of ``align`` rows (the norm chunk), so
per-chunk partial sums are identical whatever the rank count.

DA-CSR offsets are translation invariant: a rank stores its rows' offsets
and values byte-identical to the global slice and only rebases rowptr to 0.
x is held in a rank-local buffer x_ext covering global [lo, hi) =
[r0 - b, r1 + b) ∩ [0, n); the kernel reads x_ext[local_row + off +
(r0 - lo)] (the C ABI's x_offset).

Per multiply: the halo segments of x_ext are exchanged with the ranks that
own them (one NCCL send/recv group; for r1 - r0 >= b that is just the two
neighbours) while the interior rows [b, n_local - b), which need no halo,
run on the compute stream; the two boundary strips follow.

Power iteration x <- A x / ||A x||: per-chunk sums of y^2 (fixed tree),
all-gathered in rank order and folded in index order on every rank, so the
norm — and therefore every iterate — is bit-identical for 1/2/4/8 ranks.
The normalisation is folded into the next multiply's alpha.

The module is device-agnostic: the local operator is an object with
``spmv(x_ext, y, alpha, part)`` / ``partials(y)`` / ``fold(all_partials)``
(the CUDA one is ``CudaLocalOp``); tests drive it with gloo on CPU.
"""

import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


@dataclass(frozen=True)
class RowPartition:
    n: int
    bounds: tuple  # ((r0, r1), ...) per rank

    @property
    def world(self):
        return len(self.bounds)

    @classmethod
    def equal(cls, n, world, align=1):
        """Rows split as evenly as possible in units of ``align`` rows."""
        units = -(-n // align)
        cuts = [min(n, ((k * units) // world) * align) for k in range(world)] + [n]
        return cls(n, tuple((cuts[k], cuts[k + 1]) for k in range(world)))

    @classmethod
    def nnz_balanced(cls, rowptr, world, align=1):
        """row_blocks cuts (first row with rowptr >= k*nnz//world), rounded
        to the nearest ``align`` boundary, kept monotone."""
        rp = np.asarray(rowptr)
        n = len(rp) - 1
        nnz = int(rp[-1])
        cuts = [0]
        for k in range(1, world):
            b = int(np.searchsorted(rp, (k * nnz) // world, side="left"))
            b = int(round(b / align)) * align
            cuts.append(min(max(b, cuts[-1]), n))
        cuts.append(n)
        return cls(n, tuple((cuts[k], cuts[k + 1]) for k in range(world)))

    def owner_segments(self, g0, g1):
        """[(rank, s0, s1)] covering global rows [g0, g1)."""
        out = []
        for q, (a, b) in enumerate(self.bounds):
            s0, s1 = max(a, g0), min(b, g1)
            if s0 < s1:
                out.append((q, s0, s1))
        return out


@dataclass(frozen=True)
class HaloPlan:
    """What rank ``rank`` receives into / sends from its x_ext buffer."""

    rank: int
    r0: int
    r1: int
    lo: int  # global index of x_ext[0]
    hi: int
    recv: tuple  # ((peer, g0, g1), ...) halo rows owned by peer
    send: tuple  # ((peer, g0, g1), ...) own rows peer needs

    @property
    def x_offset(self):
        """Kernel x_offset: local row i, offset o -> x_ext[i + o + (r0 - lo)]."""
        return self.r0 - self.lo

    @property
    def length(self):
        return self.hi - self.lo

    def own_slice(self):
        return slice(self.r0 - self.lo, self.r1 - self.lo)


def halo_plan(part, rank, b):
    """Halo segments for a matrix of half-bandwidth ``b`` (max |col-row|)."""
    r0, r1 = part.bounds[rank]
    lo, hi = max(0, r0 - b), min(part.n, r1 + b)
    recv = [s for s in part.owner_segments(lo, r0) + part.owner_segments(r1, hi) if s[0] != rank]
    send = []
    for q, (a, c) in enumerate(part.bounds):
        if q == rank or a == c:
            continue
        qlo, qhi = max(0, a - b), min(part.n, c + b)
        for g0, g1 in ((qlo, a), (c, qhi)):
            s0, s1 = max(g0, r0), min(g1, r1)
            if s0 < s1:
                send.append((q, s0, s1))
    return HaloPlan(rank, r0, r1, lo, hi, tuple(recv), tuple(send))


def exchange_halo(x_ext, plan, group=None):
    """Fill the halo of x_ext from the owners; send own rows to who needs
    them.  One batched P2P group (NCCL: a single ncclGroupStart/End)."""
    ops = []
    for q, g0, g1 in plan.send:
        ops.append(dist.P2POp(dist.isend, x_ext[g0 - plan.lo:g1 - plan.lo], q, group))
    for q, g0, g1 in plan.recv:
        ops.append(dist.P2POp(dist.irecv, x_ext[g0 - plan.lo:g1 - plan.lo], q, group))
    if not ops:
        return []
    return dist.batch_isend_irecv(ops)


def gather_partials(p, group=None, counts=None):
    """All ranks' chunk partials concatenated in rank order.  With the
    per-rank ``counts`` known (they follow from the partition) this is one
    fixed-size all_gather; otherwise the counts are exchanged first."""
    world = dist.get_world_size(group)
    if counts is None:
        count = torch.tensor([p.numel()], dtype=torch.int64, device=p.device)
        cs = [torch.zeros_like(count) for _ in range(world)]
        dist.all_gather(cs, count, group=group)
        counts = [int(c.item()) for c in cs]
    m = max(counts)
    padded = p if p.numel() == m else torch.cat(
        [p, torch.zeros(m - p.numel(), dtype=p.dtype, device=p.device)])
    out = torch.empty(world * m, dtype=p.dtype, device=p.device)
    dist.all_gather_into_tensor(out, padded.contiguous(), group=group)
    if all(c == m for c in counts):
        return out
    return torch.cat([out[q * m:q * m + c] for q, c in enumerate(counts)])


def chunk_counts(part, chunk):
    """Norm-chunk partials per rank (rank boundaries on chunk multiples)."""
    return [-(-(b - a) // chunk) for a, b in part.bounds]


def launch_ranges(n_local, b, group=512):
    """Row ranges of a rank's three SpMV launches, interior first:
    [(cut0, cut1), (0, cut0), (cut1, n_local)].  The interior rows need no
    halo (rows >= b and < n_local - b); the cuts sit on ``group``-row
    boundaries (a few rows that need no halo join the strips) so that every
    launch covers whole 512-row groups: the TILED epilogue then returns the
    groups' sums of y^2 (no second pass over y for the norm)."""
    cut0 = min((b + group - 1) // group * group, n_local)
    cut1 = max(cut0, (n_local - b) // group * group)
    return [(cut0, cut1), (0, cut0), (cut1, n_local)]


class CudaLocalOp:
    """A rank's rows as DeviceMatrix objects (boundary strips + interior,
    each with its own plan) over one set of arrays."""

    def __init__(self, kind, rowptr, colids, values, ncols_global, plan, chunk, b,
                 variant="naive"):
        from .device import LAYOUT_KERNELS, DeviceMatrix
        from .spmv import kernel_for, resolve_variant
        n_local = rowptr.numel() - 1
        self.n_local = n_local
        self.plan = plan
        self.chunk = chunk
        self.kind = kind
        self.ranges = launch_ranges(n_local, b)
        name, order = resolve_variant(variant)
        self.order = order
        self.mats = []
        full = None
        if name == "exact" and n_local:
            # the library's selection on this rank's rows (row statistics)
            full = DeviceMatrix(kind, n_local, ncols_global, rowptr, colids, values)
            name = kernel_for(full, name, order)
        if name in LAYOUT_KERNELS and n_local:
            # one derived layout of all local rows serves the three row ranges
            if full is None:
                full = DeviceMatrix(kind, n_local, ncols_global, rowptr, colids, values)
            full.build_tiles() if name == "tiled" else full.build_slices()
            self.mats = [full if r1 > r0 else None for r0, r1 in self.ranges]
            self.kernels = [name if r1 > r0 else None for r0, r1 in self.ranges]
        else:
            for r0, r1 in self.ranges:
                dm = DeviceMatrix(kind, n_local, ncols_global, rowptr, colids, values,
                                  row_start=r0, row_end=r1) if r1 > r0 else None
                self.mats.append(dm)
            self.kernels = [kernel_for(dm, name, order) if dm is not None else None
                            for dm in self.mats]
        # CSR local colids stay global: x index = col - lo
        self.x_offset = plan.x_offset if kind == "da" else -plan.lo
        self.fused = bool(n_local) and chunk % 512 == 0 and all(
            dm is None or dm.fused_sumsq_ok(k, self.order, r0, r1)
            for dm, k, (r0, r1) in zip(self.mats, self.kernels, self.ranges))
        self.group_sumsq = (torch.empty((n_local + 511) // 512, dtype=torch.float64,
                                        device=rowptr.device) if self.fused else None)

    def spmv_part(self, which, x_ext, y, alpha, stream=None):
        dm = self.mats[which]
        if dm is not None:
            r0, r1 = self.ranges[which]
            fused = self.fused and isinstance(alpha, torch.Tensor)
            dm.spmv_into(x_ext, y, alpha, 0.0, self.kernels[which], self.order,
                         x_offset=self.x_offset, row_start=r0, row_end=r1, stream=stream,
                         group_sumsq=self.group_sumsq if fused else None)

    device_norm = True  # the norm and the next alpha stay on the device

    def partials(self, y):
        from .power import chunk_partials
        return chunk_partials(y, self.chunk).clone()

    def partials_after_spmv(self, y):
        """The chunk partials of the y the three spmv_part launches just
        wrote (device alpha): from their fused group sums when available."""
        if not self.fused:
            return self.partials(y)
        from .power import partials_from_groups
        return partials_from_groups(self.group_sumsq, self.n_local, self.chunk).clone()

    def fold(self, allp):
        from .power import fold_ordered
        return float(fold_ordered(allp).item())

    def norm_alpha(self, allp, norm_out, alpha_out):
        from .power import norm_alpha
        norm_alpha(allp, norm_out, alpha_out)

    def scale(self, x, factor):
        from .power import scale_by_device_factor
        scale_by_device_factor(x, factor)


def dist_spmv(op, x_ext, y, alpha, plan, group=None, overlap=True):
    """y = alpha * A_local x (x_ext's own rows current, halo exchanged here).

    CUDA: the interior rows run on the current stream while the halo is in
    flight on NCCL's stream; the two boundary strips run on a side stream
    that waits only for the exchange, so they overlap the interior's tail."""
    if overlap and x_ext.is_cuda:
        cur = torch.cuda.current_stream(x_ext.device)
        side = getattr(op, "side_stream", None)
        if side is None:
            side = op.side_stream = torch.cuda.Stream(x_ext.device)
        side.wait_stream(cur)                      # x_ext / y ready for the strips
        reqs = exchange_halo(x_ext, plan, group)   # NCCL stream
        op.spmv_part(0, x_ext, y, alpha)           # interior: no halo needed
        with torch.cuda.stream(side):
            for r in reqs:
                r.wait()                           # side stream waits on NCCL
            op.spmv_part(1, x_ext, y, alpha, stream=side)
            op.spmv_part(2, x_ext, y, alpha, stream=side)
        cur.wait_stream(side)
    else:
        for r in exchange_halo(x_ext, plan, group):
            r.wait()
        for which in range(3):
            op.spmv_part(which, x_ext, y, alpha)
    return y


def power_iteration(op, plan, x0_own, iters, group=None, overlap=True, counts=None):
    """Distributed normalised power iteration from x0 (this rank's rows).

    Returns (x_own, norms): x_own = x_iters restricted to this rank's rows,
    norms[k] = ||A x_k||.  Identical bits for every rank count.  ``counts``:
    the per-rank number of norm chunks (chunk_counts), which makes each norm
    one fixed-size all_gather.
    """
    dev = x0_own.device
    bufs = [torch.zeros(plan.length, dtype=x0_own.dtype, device=dev) for _ in range(2)]
    own = plan.own_slice()
    bufs[0][own] = x0_own
    if getattr(op, "device_norm", False) and counts is not None:
        # no host round trip: alpha and the norms live on the device
        alpha = torch.empty(1, dtype=torch.float64, device=dev)
        norms = torch.empty(iters + 1, dtype=torch.float64, device=dev)
        op.norm_alpha(gather_partials(op.partials(x0_own), group, counts), norms[0:1], alpha)
        cur = 0
        for k in range(iters):
            nxt = 1 - cur
            dist_spmv(op, bufs[cur], bufs[nxt][own], alpha, plan, group, overlap)
            after = getattr(op, "partials_after_spmv", op.partials)
            op.norm_alpha(gather_partials(after(bufs[nxt][own]), group, counts),
                          norms[k + 1:k + 2], alpha)
            cur = nxt
        x = bufs[cur][own].clone()
        op.scale(x, alpha)
        return x, norms[1:].tolist()
    s_prev = math.sqrt(op.fold(gather_partials(op.partials(x0_own), group, counts)))
    norms = []
    cur = 0
    for _ in range(iters):
        nxt = 1 - cur
        dist_spmv(op, bufs[cur], bufs[nxt][own], 1.0 / s_prev, plan, group, overlap)
        s_prev = math.sqrt(op.fold(gather_partials(op.partials(bufs[nxt][own]), group, counts)))
        norms.append(s_prev)
        cur = nxt
    x = bufs[cur][own].clone()
    x.mul_(1.0 / s_prev) if not x.is_cuda else _scale_device(x, 1.0 / s_prev)
    return x, norms


def _scale_device(x, s):
    import ctypes
    from . import _native
    from .device import _stream_ptr
    _native.check(_native.lib().dacsr_scale(ctypes.c_void_p(x.data_ptr()),
                                            _native.dtype_code(x.dtype), x.numel(), s,
                                            _stream_ptr(None)), "dacsr_scale")


# ------------------------------------------------------------------ bench
def _peak_gbs():
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0


def iterate_digest(x_own, r0, chunk, group=None):
    """Partition-independent SHA-256 of the global iterate: per-chunk digests
    of this rank's rows (rank boundaries are chunk multiples), gathered in
    chunk order on every rank, hashed once more."""
    import hashlib
    xh = x_own.cpu().numpy()
    digs = [hashlib.sha256(xh[i:i + chunk].tobytes()).digest() for i in range(0, len(xh), chunk)]
    mine = torch.tensor(np.frombuffer(b"".join(digs), dtype=np.uint8).copy())
    world = dist.get_world_size(group)
    sizes = [None] * world
    dist.all_gather_object(sizes, (r0, mine.numel()), group=group)
    allb = [None] * world
    dist.all_gather_object(allb, bytes(mine.numpy()), group=group)
    order = sorted(range(world), key=lambda q: sizes[q][0])
    return hashlib.sha256(b"".join(allb[q] for q in order)).hexdigest()


def bench_main(args, rank, world, local):
    """Config C5 at N ranks (strong scaling): 50 normalised power iterations
    x <- A x / ||A x|| on the 2^28-row band (b = 32767, clip(Poisson(8), 1,
    32), DA-CSR i16, f64).  Rows in equal contiguous blocks aligned to the
    2^16-row norm chunk; each rank generates its rows on its GPU (identical
    to the same rows of the whole matrix), runs the library's default kernel
    for them (row statistics -> TILED) with the +-b halo exchanged over NCCL
    while the interior rows run, and folds the norm from one fixed-size
    all_gather of chunk partials.  One step = the 50 iterations; max over
    ranks of CUDA-event step times."""
    import json
    import time
    from .gen import banded_arrays, normal_vector
    from .harness import ClockSampler
    from .model import StorageWidths, spmv_traffic
    from .workloads import BANDED_CONFIGS

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # a failed or hung collective aborts the communicator and raises in
    # every rank (instead of blocking the stream for ever); the watchdog's
    # limit is generous against the matrix build and tight against a hang
    import datetime
    import os
    os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "1")
    dist.init_process_group(
        "nccl", device_id=dev,
        timeout=datetime.timedelta(seconds=int(os.environ.get("DACSR_NCCL_TIMEOUT_S", "600"))))
    n, b, lam, kmax, seed = BANDED_CONFIGS["c5"]
    chunk = 1 << 16
    iters = 50
    part = RowPartition.equal(n, world, align=chunk)
    plan = halo_plan(part, rank, b)
    counts = chunk_counts(part, chunk)
    r0, r1 = part.bounds[rank]
    t0 = time.time()
    arr = banded_arrays(n, b, lam, kmax, seed, dev, r0=r0, r1=r1, kinds=("da",))
    op = CudaLocalOp("da", arr["rowptr"], arr["offsets"], arr["values"], n, plan, chunk, b)
    x0 = normal_vector(r1 - r0, 21, dev, i0=r0)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    nnz_local = torch.tensor([arr["nnz"]], dtype=torch.int64, device=dev)
    dist.all_reduce(nnz_local)
    nnz = int(nnz_local.item())
    # whole-job algorithmic bytes per SpMV: the 1-GPU model of the whole
    # matrix (rowptr counted at int32, as every rank stores it)
    traffic = spmv_traffic(n, n, nnz, StorageWidths(4, 2, 8)).total_bytes
    for _ in range(max(1, args.warmup)):
        power_iteration(op, plan, x0, 2, counts=counts)
    torch.cuda.synchronize()
    dist.barrier()
    times = []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            x, norms = power_iteration(op, plan, x0, iters, counts=counts)
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
    t = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total = float(t.item())
    step = total / args.steps
    value = iters * traffic / step / 1e9
    digest = iterate_digest(x, r0, chunk)

    # e2e: host buffers through the same path — every SpMV copies this
    # rank's x rows in from pinned memory and its y rows out; max over ranks
    e2e_spmv, e2e_steps = 2, 2
    own = plan.own_slice()
    bufs = [torch.zeros(plan.length, dtype=torch.float64, device=dev) for _ in range(2)]
    xh = torch.empty(r1 - r0, dtype=torch.float64, pin_memory=True)
    yh = torch.empty(r1 - r0, dtype=torch.float64, pin_memory=True)
    xh.copy_(x0.cpu())
    dist.barrier()
    torch.cuda.synchronize()
    tt = time.perf_counter()
    for _ in range(e2e_steps):
        for _ in range(e2e_spmv):
            bufs[0][own].copy_(xh, non_blocking=True)
            dist_spmv(op, bufs[0], bufs[1][own], 1.0, plan)
            yh.copy_(bufs[1][own], non_blocking=True)
            torch.cuda.current_stream().synchronize()
    el = torch.tensor([time.perf_counter() - tt], dtype=torch.float64, device=dev)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    e2e_gbs = e2e_steps * e2e_spmv * traffic / float(el.item()) / 1e9
    if rank == 0:
        line = {
            "metric": "SpMV effective HBM GB/s (DA-CSR i16, f64)", "value": round(value, 1),
            "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * step, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C5: 50 normalised power iterations, banded n=2^28, b=32767, "
                                   "clip(Poisson(8),1,32), DA-CSR i16 f64",
                       "nnz": nnz, "bytes_per_spmv": traffic, "iters_per_step": iters,
                       "parallelism": f"row blocks x{world}, +-{b}-row halo (NCCL send/recv "
                                      "overlapped with the interior rows), norm: sums of "
                                      "y^2 by 512-row groups out of the SpMV epilogue"
                                      + ("" if op.fused else " (not fused here)") +
                                      ", one all_gather of 2^16-row chunk partials",
                       "kernel": op.kernels[0], "build_s": round(build_s, 1),
                       "final_norm": norms[-1],
                       "iterate_sha256": digest,
                       "note": "final_norm and iterate_sha256 are identical for every rank "
                               "count (deterministic chunked norm)"},
            "roofline": {"bound": "hbm", "achieved": round(value / world, 1),
                         "peak": _peak_gbs(), "unit": "GB/s",
                         "frac": round(value / world / _peak_gbs(), 4), "traffic": None,
                         "note": "per GPU: whole-job model bytes / N / max-over-ranks step time"},
            "e2e": {"value": round(e2e_gbs, 1), "unit": "GB/s",
                    "h2d_bytes_per_step": e2e_spmv * n * 8, "d2h_bytes_per_step": e2e_spmv * n * 8,
                    "spmv_per_step": e2e_spmv,
                    "note": "each rank: pinned host x rows -> distributed SpMV -> host y rows"},
            "gpu_launches": args.steps * iters * 5,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
