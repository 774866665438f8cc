"""Normalised power iteration x <- A x / ||A x||_2 (config C5) on one GPU.

The norm is deterministic: ``dacsr_sumsq_chunks`` reduces y^2 over fixed
row chunks with a fixed tree, ``dacsr_sum_ordered`` folds the chunk
partials in index order.  With rank boundaries on chunk boundaries the
multi-GPU run (distributed.py) folds the very same partials, so 1/2/4/8
GPUs produce bit-identical iterates.  The normalisation is folded into the
next SpMV's alpha (y_k = (1/s_{k-1}) * A y_{k-1}), i.e. the reference API's
own ``alpha`` argument, so the CPU oracle replays it exactly.
"""

import ctypes
import math

import torch

from . import _native
from .device import _stream_ptr

DEFAULT_CHUNK = 1 << 16


def chunk_partials(y, chunk=DEFAULT_CHUNK, stream=None, out=None):
    """Per-chunk sums of y^2 (device float64 tensor of ceil(n/chunk))."""
    n = y.numel()
    m = (n + chunk - 1) // chunk
    if out is None:
        out = torch.empty(max(m, 1), dtype=torch.float64, device=y.device)
    _native.check(_native.lib().dacsr_sumsq_chunks(
        ctypes.c_void_p(y.data_ptr()), _native.dtype_code(y.dtype), n, chunk,
        ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)), "dacsr_sumsq_chunks")
    return out[:m]


def fold_ordered(partials, stream=None, out=None):
    """Sum of partials in index order (device float64 scalar tensor)."""
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=partials.device)
    _native.check(_native.lib().dacsr_sum_ordered(
        ctypes.c_void_p(partials.data_ptr()), partials.numel(), ctypes.c_void_p(out.data_ptr()),
        _stream_ptr(stream)), "dacsr_sum_ordered")
    return out


def chunked_sumsq(y, chunk=DEFAULT_CHUNK, stream=None):
    out = fold_ordered(chunk_partials(y, chunk, stream), stream)
    if stream is not None:
        stream.synchronize()  # .item() reads on the current stream
    return float(out.item())


def power_iteration(dm, x0, iters=50, chunk=DEFAULT_CHUNK, variant="naive", order=0,
                    stream=None):
    """Run ``iters`` normalised power steps from x0 (device tensor).

    ``variant``: a kernel name, or a reference variant name ("naive", ...)
    resolved by the library's selection for this matrix.

    Returns (x, norms) with norms[k] = ||A x_k|| and x = x_iters.
    x_0 = x0 / ||x0||; y_k = alpha_k * A y_{k-1} with alpha_k = 1/s_{k-1}
    (alpha_0 = 1/||x0||, y_{-1} = x0); s_k = ||y_k||; x_iters = y/s.
    """
    from .spmv import _EXACT, kernel_for, resolve_variant
    if variant in _EXACT or variant == "auto":
        name, order = resolve_variant(variant)
        variant = kernel_for(dm, name, order)
    bufs = [x0.clone(), torch.empty_like(x0)]
    s_prev = math.sqrt(chunked_sumsq(x0, chunk, stream))
    norms = []
    cur = 0
    for _ in range(iters):
        alpha = 1.0 / s_prev
        dm.spmv_into(bufs[cur], bufs[1 - cur], alpha, 0.0, variant, order, stream=stream)
        cur = 1 - cur
        s_prev = math.sqrt(chunked_sumsq(bufs[cur], chunk, stream))
        norms.append(s_prev)
    x = bufs[cur]
    _native.check(_native.lib().dacsr_scale(
        ctypes.c_void_p(x.data_ptr()), _native.dtype_code(x.dtype), x.numel(), 1.0 / s_prev,
        _stream_ptr(stream)), "dacsr_scale")
    return x, norms
