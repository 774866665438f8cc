"""TEST INFRASTRUCTURE ONLY — Python face of the CPU oracle.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` arm may import this module, and only as the checker or
the timed CPU baseline.  The product package never imports it.

What it restates (file:line into /root/reference/pkg/src/dacsr):
* ``spmv``          spmv/__init__.py:104-183 semantics (alpha==0 short-cut at
                    150-156) over the C kernels in dacsr_oracle.c
                    (_numba_kernels.py:12-160)
* ``row_blocks``    spmv/__init__.py:71-85 (C)
* ``bandwidth`` / ``dacsr_offsets``   core.py:320-355 (numpy)
* ``symmetrized_adjacency``           reorder.py:70-97 (numpy)
* ``rcm``           reorder.py:146-197 (C)
* ``permute``       reorder.py:200-220 with core.py:270-301 (numpy)
* ``time_kernel``   bench.py:96-115
* the C3/C5 banded generator restatement (gen_oracle.c)

Pinned against tests/golden/ (made by the reference itself) in
tests/test_oracle.py.
"""

import ctypes
import math
import os
import subprocess
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

ORDERS = {"naive": 0, "shifted_base": 0, "multi_accumulator_3": 1, "strip_mined_4": 2}
_DT = {np.dtype(np.int8): 0, np.dtype(np.int16): 1, np.dtype(np.int32): 2,
       np.dtype(np.int64): 3, np.dtype(np.float32): 4, np.dtype(np.float64): 5,
       np.dtype(np.float16): 6}
BF16 = 7  # bfloat16 arrays travel as uint16 bit patterns (numpy has no bf16)

_lib = None


def build():
    """Compile liboracle.so (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32, d, u64 = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                ctypes.c_double, ctypes.c_uint64)
        L.orc_spmv.argtypes = [i32] * 5 + [vp] * 5 + [d, d, i64, i64]
        L.orc_spmv_parallel.argtypes = [i32] * 5 + [vp] * 5 + [d, d, i64, i32]
        L.orc_row_blocks.argtypes = [vp, i32, i64, i64, vp]
        L.orc_to_half_bits.argtypes = [vp, vp, i64, i32]
        L.orc_from_half_bits.argtypes = [vp, vp, i64, i32]
        L.orc_rcm.argtypes = [i64, vp, vp, vp]
        L.orc_gen_row.argtypes = [i64, i64, i32, u64, vp, i64, vp]
        L.orc_gen_value.argtypes = [i64, u64, i64, ctypes.c_int32, vp]
        L.orc_gen_value.restype = d
        L.orc_gen_counts.argtypes = [i64, i64, i32, u64, vp, i64, i64, vp]
        L.orc_gen_fill.argtypes = [i64, i64, i32, u64, vp, vp, i64, i64, vp, vp]
        L.orc_gen_fill.restype = i64
        L.orc_gen_normal.argtypes = [u64, i64, i64, vp, vp]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _rowptr_arg(rowptr):
    rp = np.ascontiguousarray(rowptr)
    if rp.dtype not in (np.int32, np.int64):
        rp = rp.astype(np.int64)
    return rp


def to_half_bits(a, bf16=False):
    """float64 array -> 16-bit patterns (binary16 or bfloat16), one RNE rounding."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    out = np.empty(a.shape, np.uint16)
    lib().orc_to_half_bits(_p(a), _p(out), a.size, int(bf16))
    return out


def from_half_bits(bits, bf16=False):
    """16-bit patterns -> float64 (exact)."""
    b = np.ascontiguousarray(bits).view(np.uint16)
    out = np.empty(b.shape, np.float64)
    lib().orc_from_half_bits(_p(b), _p(out), b.size, int(bf16))
    return out


def spmv_kernel(kind, rowptr, colids, values, x, y, alpha, beta, order="naive",
                row_start=0, row_end=None, threads=1, x_offset=0, bf16=False):
    """Run the restated reference kernel in place on ``y``.

    ``kind`` is "csr" or "da"; ``threads > 1`` is ParallelRowBlock(threads).
    ``x_offset`` shifts x addressing (x[col + x_offset]) for rank-local halo
    buffers; the reference kernel is the x_offset == 0 case.  16-bit values
    (an extension, no reference kernel): float16 arrays, or with ``bf16``
    uint16 arrays holding bfloat16 bit patterns.
    """
    rp = _rowptr_arg(rowptr)
    ci = np.ascontiguousarray(colids)
    v = np.ascontiguousarray(values)
    xx = np.ascontiguousarray(x)
    assert y.flags.c_contiguous and y.dtype == v.dtype == xx.dtype
    nrows = len(rp) - 1
    row_end = nrows if row_end is None else row_end
    k = {"csr": 0, "da": 1}[kind]
    xp = ctypes.c_void_p((xx.ctypes.data or 0) + int(x_offset) * xx.itemsize)
    vcode = BF16 if bf16 else _DT[v.dtype]
    args = (k, ORDERS[order], _DT[rp.dtype], _DT[ci.dtype], vcode,
            _p(rp), _p(ci), _p(v), xp, _p(y), float(alpha), float(beta))
    if threads == 1:
        rc = lib().orc_spmv(*args, row_start, row_end)
    else:
        assert row_start == 0 and row_end == nrows
        rc = lib().orc_spmv_parallel(*args, nrows, threads)
    if rc:
        raise RuntimeError(f"oracle spmv failed ({rc})")
    return y


def spmv(kind, rowptr, colids, values, x, y=None, alpha=1.0, beta=0.0, order="naive",
         threads=1):
    """Reference ``spmv`` semantics (spmv/__init__.py:128-183) on the oracle."""
    alpha, beta = float(alpha), float(beta)
    nrows = len(rowptr) - 1
    if y is None:
        assert beta == 0.0
        y = np.empty(nrows, dtype=values.dtype)
    if alpha == 0.0:
        if beta == 0.0:
            y[:] = 0.0
        elif beta != 1.0:
            y[:] = np.float64(beta) * y
        return y
    return spmv_kernel(kind, rowptr, colids, values, x, y, alpha, beta, order,
                       threads=threads)


def row_blocks(rowptr, nblocks):
    rp = _rowptr_arg(rowptr)
    cuts = np.empty(nblocks + 1, dtype=np.int64)
    if lib().orc_row_blocks(_p(rp), _DT[rp.dtype], len(rp) - 1, nblocks, _p(cuts)):
        raise ValueError("nblocks must be >= 1")
    return [(int(cuts[i]), int(cuts[i + 1])) for i in range(nblocks)]


def entry_rows(rowptr):
    rp = np.asarray(rowptr, dtype=np.int64)
    return np.repeat(np.arange(len(rp) - 1, dtype=np.int64), np.diff(rp))


def bandwidth_csr(rowptr, colids):
    if len(colids) == 0:
        return 0
    return int(np.abs(np.asarray(colids, np.int64) - entry_rows(rowptr)).max())


def dacsr_offsets(rowptr, colids, bits=16):
    """(offsets, ok): col - row cast to int-bits, ok=False when w too large."""
    w = bandwidth_csr(rowptr, colids)
    if w > 2 ** (bits - 1) - 1:
        return None, False
    off = np.asarray(colids, np.int64) - entry_rows(rowptr)
    return off.astype({8: np.int8, 16: np.int16, 32: np.int32, 64: np.int64}[bits]), True


def symmetrized_adjacency(n, rowptr, colids):
    """Pattern of A + A^T without self loops, sorted and deduplicated."""
    rows = entry_rows(rowptr)
    cols = np.asarray(colids, np.int64)
    keep = rows != cols
    u = np.concatenate([rows[keep], cols[keep]])
    v = np.concatenate([cols[keep], rows[keep]])
    order = np.lexsort((v, u))
    u, v = u[order], v[order]
    if len(u):
        first = np.ones(len(u), dtype=bool)
        first[1:] = (u[1:] != u[:-1]) | (v[1:] != v[:-1])
        u, v = u[first], v[first]
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(u, minlength=n), out=indptr[1:])
    return indptr, np.ascontiguousarray(v, dtype=np.int64)


def rcm(n, rowptr, colids):
    """perm[new] = old, the reference's reverse Cuthill–McKee order."""
    indptr, indices = symmetrized_adjacency(n, rowptr, colids)
    perm = np.empty(n, dtype=np.int64)
    if lib().orc_rcm(n, _p(indptr), _p(indices), _p(perm)):
        raise MemoryError("oracle rcm allocation failed")
    return perm


def permute(n, rowptr, colids, values, perm):
    """(rowptr, colids, values) of P A P^T, canonical, widths preserved."""
    perm = np.asarray(perm, np.int64)
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n, dtype=np.int64)
    r = inv[entry_rows(rowptr)]
    c = inv[np.asarray(colids, np.int64)]
    order = np.lexsort((c, r))
    r, c = r[order], c[order]
    v = np.asarray(values)[order]
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=rp[1:])
    return (rp.astype(np.asarray(rowptr).dtype), c.astype(np.asarray(colids).dtype), v)


def time_kernel(fn, epochs=11, warmup_iters=10, min_epoch_iters=10, min_epoch_time=0.1,
                clock=time.perf_counter):
    """Best-of-epochs per-iteration seconds (bench.py:96-115)."""
    for _ in range(warmup_iters):
        fn()
    best = math.inf
    for _ in range(epochs):
        iters = 0
        t0 = clock()
        while True:
            fn()
            iters += 1
            el = clock() - t0
            if iters >= min_epoch_iters and el >= min_epoch_time:
                break
        best = min(best, el / iters)
    return best


# ---- C3/C5 generator restatement -----------------------------------------

def gen_row(n, b, kmax, seed, cdf, r):
    offs = np.empty(128, np.int32)
    m = lib().orc_gen_row(n, b, kmax, seed, _p(cdf), r, _p(offs))
    return offs[:m].copy()


def gen_value(b, seed, r, off, table):
    return lib().orc_gen_value(b, seed, r, int(off), _p(table))


def gen_counts(n, b, kmax, seed, cdf, r0, r1):
    if kmax - 1 > 2 * b:
        raise ValueError("kmax - 1 distinct non-zero offsets do not exist in [-b, b]")
    out = np.empty(r1 - r0, np.int32)
    lib().orc_gen_counts(n, b, kmax, seed, _p(cdf), r0, r1, _p(out))
    return out


def gen_fill(n, b, kmax, seed, cdf, table, r0=0, r1=None):
    """Full (rowptr i64, offsets i16, values f64) of rows [r0, r1)."""
    r1 = n if r1 is None else r1
    counts = gen_counts(n, b, kmax, seed, cdf, r0, r1)
    rp = np.zeros(r1 - r0 + 1, np.int64)
    np.cumsum(counts, out=rp[1:])
    offs = np.empty(int(rp[-1]), np.int16)
    vals = np.empty(int(rp[-1]), np.float64)
    got = lib().orc_gen_fill(n, b, kmax, seed, _p(cdf), _p(table), r0, r1, _p(offs), _p(vals))
    assert got == rp[-1]
    return rp, offs, vals


def gen_fill_parallel(n, b, kmax, seed, cdf, table, r0=0, r1=None, threads=None):
    """gen_fill over row blocks on host threads (ctypes releases the GIL);
    identical arrays (rows are pure functions of (seed, row))."""
    import concurrent.futures as cf
    import os
    r1 = n if r1 is None else r1
    threads = threads or len(os.sched_getaffinity(0))
    cuts = np.linspace(r0, r1, threads * 4 + 1).astype(np.int64)
    blocks = [(int(a), int(c)) for a, c in zip(cuts[:-1], cuts[1:]) if c > a]
    with cf.ThreadPoolExecutor(threads) as ex:
        parts = list(ex.map(lambda bc: gen_counts(n, b, kmax, seed, cdf, *bc), blocks))
    counts = np.concatenate(parts) if parts else np.zeros(0, np.int32)
    rp = np.zeros(r1 - r0 + 1, np.int64)
    np.cumsum(counts, out=rp[1:])
    offs = np.empty(int(rp[-1]), np.int16)
    vals = np.empty(int(rp[-1]), np.float64)

    def fill(bc):
        a, c = bc
        e0 = int(rp[a - r0])
        po = ctypes.c_void_p(offs.ctypes.data + 2 * e0)
        pv = ctypes.c_void_p(vals.ctypes.data + 8 * e0)
        got = lib().orc_gen_fill(n, b, kmax, seed, _p(cdf), _p(table), a, c, po, pv)
        assert got == rp[c - r0] - rp[a - r0]

    with cf.ThreadPoolExecutor(threads) as ex:
        list(ex.map(fill, blocks))
    return rp, offs, vals


def gen_normal(seed, i0, i1, table):
    out = np.empty(i1 - i0, np.float64)
    lib().orc_gen_normal(seed, i0, i1, _p(table), _p(out))
    return out


# ---- deterministic norm restatement (csrc/aux.cu sumsq_kernel) -----------

def sumsq_chunks(y, chunk):
    """Per-chunk sum of y^2 in the device's fixed GROUP TREE (csrc/aux.cu
    group_sumsq, also the TILED kernel's fused epilogue): a chunk is cut into
    groups of 512 values from its start; in a group lane l folds
    sq(y[32j + l]), j = 0..15 in order (values past the end are skipped:
    adding +0.0 to a sum that started at +0.0 changes nothing), a 5-step xor
    butterfly over the 32 lanes gives the group sum, and the chunk's partial
    is its group sums folded left to right."""
    y = np.asarray(y, dtype=np.float64)
    n = len(y)
    out = []
    lanes = np.arange(32)
    for c0 in range(0, n, chunk):
        seg = y[c0:min(n, c0 + chunk)]
        ng = (len(seg) + 511) // 512
        pad = np.zeros(ng * 512)
        pad[:len(seg)] = seg
        sq = (pad * pad).reshape(ng, 16, 32)
        acc = np.zeros((ng, 32))
        for j in range(16):
            acc = acc + sq[:, j, :]
        for o in (16, 8, 4, 2, 1):
            acc = acc + acc[:, lanes ^ o]
        t = 0.0
        for v in acc[:, 0].tolist():
            t = t + v
        out.append(t)
    return np.array(out)


def fold_ordered(partials):
    t = 0.0
    for v in np.asarray(partials, dtype=np.float64).tolist():
        t = t + v
    return t
