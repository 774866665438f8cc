"""Normalised power iteration x <- A x / ||A x||_2 (config C5) on one GPU.

The norm is deterministic: ``dacsr_sumsq_chunks`` reduces y^2 over fixed
row chunks with a fixed tree (512-row groups: 16 values per lane, an xor
butterfly, the groups left to right), ``dacsr_sum_ordered`` folds the chunk
partials in index order.  The TILED SpMV produces the same group sums in its
epilogue (``spmv_into(group_sumsq=...)``), so an iteration does not read y a
second time.  With rank boundaries on chunk boundaries the
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


def partials_from_groups(group_sumsq, n, chunk=DEFAULT_CHUNK, stream=None, out=None):
    """Per-chunk sums of y^2 from the 512-row group sums a fused SpMV stored
    (DeviceMatrix.spmv_into(group_sumsq=...)): the very partials
    ``chunk_partials`` computes from y, without reading y again."""
    m = (n + chunk - 1) // chunk
    if out is None:
        out = torch.empty(max(m, 1), dtype=torch.float64, device=group_sumsq.device)
    _native.check(_native.lib().dacsr_sumsq_from_groups(
        ctypes.c_void_p(group_sumsq.data_ptr()), n, chunk, ctypes.c_void_p(out.data_ptr()),
        _stream_ptr(stream)), "dacsr_sumsq_from_groups")
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


def norm_alpha(partials, norm_out, alpha_out, stream=None):
    """On the device: s = sqrt(ordered fold of partials), norm_out[0] = s,
    alpha_out[0] = 1 / s (Python's math.sqrt and 1.0 / s, bit for bit)."""
    _native.check(_native.lib().dacsr_norm_alpha(
        ctypes.c_void_p(partials.data_ptr()), partials.numel(),
        ctypes.c_void_p(norm_out.data_ptr()) if norm_out is not None else None,
        ctypes.c_void_p(alpha_out.data_ptr()), _stream_ptr(stream)), "dacsr_norm_alpha")


def scale_by_device_factor(x, factor, stream=None):
    """x *= factor[0] (factor a float64 device scalar), one rounding."""
    _native.check(_native.lib().dacsr_scale_dev(
        ctypes.c_void_p(x.data_ptr()), _native.dtype_code(x.dtype), x.numel(),
        ctypes.c_void_p(factor.data_ptr()), _stream_ptr(stream)), "dacsr_scale_dev")


class PowerIteration:
    """``iters`` normalised power steps on one GPU, entirely on the device:
    each step is the SpMV with alpha read from device memory
    (dacsr_spmv_dev_alpha), the chunked sum of squares of the result and the
    norm / next alpha (dacsr_norm_alpha) — no host round trip, so the whole
    run can be captured once in a CUDA graph and replayed.

    Semantics (identical to the host loop it replaced): x_0 = x0 / ||x0||;
    y_k = alpha_k * A y_{k-1} with alpha_k = 1/s_{k-1} (alpha_0 = 1/||x0||,
    y_{-1} = x0); s_k = ||y_k||; the result is y / s.
    """

    def __init__(self, dm, x0, iters=50, chunk=DEFAULT_CHUNK, variant="naive", order=0,
                 graph=False):
        from .spmv import _EXACT, kernel_for, resolve_variant
        if variant in _EXACT or variant == "auto":
            name, order = resolve_variant(variant)
            variant = kernel_for(dm, name, order)
        self.dm, self.iters, self.chunk, self.variant, self.order = dm, iters, chunk, variant, order
        self.x0 = x0
        self.bufs = [torch.empty_like(x0), torch.empty_like(x0)]
        dev = x0.device
        m = (x0.numel() + chunk - 1) // chunk
        self.partials = torch.empty(max(m, 1), dtype=torch.float64, device=dev)
        self.alpha = torch.empty(1, dtype=torch.float64, device=dev)
        self.norms = torch.empty(iters + 1, dtype=torch.float64, device=dev)
        # ||y||^2 out of the SpMV's own epilogue where the kernel offers it
        # (TILED, whole 512-row groups): no second pass over y
        self.fused = (chunk % 512 == 0 and dm.nrows == x0.numel()
                      and dm.fused_sumsq_ok(variant, order))
        self.group_sumsq = (torch.empty((x0.numel() + 511) // 512, dtype=torch.float64, device=dev)
                            if self.fused else None)
        self.graph = None
        if graph:
            self._launch()  # warm: derived layout, launch-config caches
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            with torch.cuda.graph(g, stream=s):
                self._launch()
            torch.cuda.synchronize()
            self.graph = g

    def _launch(self, stream=None):
        dm, chunk = self.dm, self.chunk
        self.bufs[0].copy_(self.x0)
        chunk_partials(self.bufs[0], chunk, stream, out=self.partials)
        norm_alpha(self.partials, self.norms[0:1], self.alpha, stream)
        cur = 0
        for k in range(self.iters):
            dm.spmv_into(self.bufs[cur], self.bufs[1 - cur], self.alpha, 0.0, self.variant,
                         self.order, stream=stream, group_sumsq=self.group_sumsq)
            cur = 1 - cur
            if self.fused:
                partials_from_groups(self.group_sumsq, self.x0.numel(), chunk, stream,
                                     out=self.partials)
            else:
                chunk_partials(self.bufs[cur], chunk, stream, out=self.partials)
            norm_alpha(self.partials, self.norms[k + 1:k + 2], self.alpha, stream)
        self.cur = cur

    def run(self):
        """Enqueue the whole run (graph replay when captured); returns x."""
        if self.graph is not None:
            self.graph.replay()
            self.cur = self.iters % 2
        else:
            self._launch()
        return self.bufs[self.cur]

    def result(self):
        """(x_iters, norms) after run(): x = y / s (a copy), norms on the host."""
        x = self.bufs[self.cur].clone()
        scale_by_device_factor(x, self.alpha)
        return x, self.norms[1:].tolist()


def power_iteration(dm, x0, iters=50, chunk=DEFAULT_CHUNK, variant="naive", order=0,
                    stream=None):
    """Run ``iters`` normalised power steps from x0 (device tensor); returns
    (x, norms) with norms[k] = ||A x_k|| (see PowerIteration)."""
    with torch.cuda.stream(stream) if stream is not None else _nullctx():
        pi = PowerIteration(dm, x0, iters, chunk, variant, order)
        pi.run()
        return pi.result()


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False
