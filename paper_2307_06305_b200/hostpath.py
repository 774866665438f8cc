"""Streamed host path: ``spmv(A, x_host, y_host)`` with the copies overlapped.

A row block [r0, r1) of a matrix of bandwidth w only reads x[r0 - w, r1 + w).
So the call is split into P row pieces on three streams:

    h2d  : x[0 : r1_p + w]  (only the part not sent yet), y piece if beta != 0
    comp : waits for its x/y prefix, runs the SpMV kernel on rows [r0_p, r1_p)
    d2h  : waits for the piece's kernel, copies y[r0_p : r1_p] back

The H2D of later pieces, the kernels and the D2H of earlier pieces overlap
(PCIe/C2C is full duplex), so for a banded operator the call costs about
max(bytes(x), bytes(y)) / link bandwidth instead of their sum.  Results are
bit-identical to the one-shot path: each row is computed by the same kernel
with the same exact order (each piece is a row range with its own plan).
"""

import numpy as np
import torch

from .device import LAYOUT_KERNELS
from .spmv import kernel_for


class StreamedHost:
    """Per-DeviceMatrix resources of the streamed host path (cached)."""

    def __init__(self, dm, pieces=None, cuts=None, y_through_device=None):
        # pieces: equal row pieces (C2: 1 -> 0.72 ms, 4 -> 0.61 ms, 16 -> 0.93 ms;
        # C3, 134 MB of x and of y: 4 -> 3.77 ms, 8 -> 3.55 ms with y returned by
        # the copy engine, 3.72 ms with the kernels storing it over the link,
        # 16 -> 3.62 / 4.06 ms: tools/e2e_c3_pieces.py);
        # cuts: interior cut points as row fractions instead (small first and
        # last pieces shorten the pipeline fill and drain)
        from .device import DeviceMatrix, bandwidth_device
        self.dm = dm
        n = dm.nrows
        big = (dm.row_end - dm.row_start) * dm.values.element_size() >= (64 << 20)
        if pieces is None:
            pieces = 8 if big else 4
        self.y_through_device = int(big if y_through_device is None else y_through_device)
        self.w = bandwidth_device(dm) if dm.nnz else 0
        if cuts is None:
            cuts = np.linspace(dm.row_start, dm.row_end, pieces + 1).astype(np.int64)
        else:
            span = dm.row_end - dm.row_start
            cuts = np.array([dm.row_start] + [dm.row_start + int(f * span) for f in cuts]
                            + [dm.row_end], dtype=np.int64)
        self.views = []
        for r0, r1 in zip(cuts[:-1], cuts[1:]):
            if r1 > r0:
                v = DeviceMatrix(dm.kind, n, dm.ncols, dm.rowptr, dm.colids, dm.values,
                                 row_start=int(r0), row_end=int(r1))
                self.views.append(v)
        dev = dm.device
        self.x = torch.empty(max(dm.ncols, 1), dtype=dm.values.dtype, device=dev)
        self.y = torch.empty(max(n, 1), dtype=dm.values.dtype, device=dev)
        self._plans = {}
        self.s_h2d = torch.cuda.Stream(dev)
        self.s_comp = torch.cuda.Stream(dev)
        self.s_d2h = torch.cuda.Stream(dev)

    def run(self, x_host, y_host, alpha, beta, kname, order):
        """One C-ABI call issues every copy, event and kernel of the pipeline
        (dacsr_spmv_host_streamed); Python only resolves the per-piece plans
        once per (kernel, order)."""
        import ctypes
        from . import _native
        key = (kname, order)
        rec = self._plans.get(key)
        if rec is None:
            k = kernel_for(self.dm, kname, order)
            plans = (_native.Plan * len(self.views))()
            if k in LAYOUT_KERNELS:
                # the pieces share the whole matrix's derived layout (the
                # kernel takes any row range inside it); no row-block table
                pl = self.dm.plan_for(k)
                for i, v in enumerate(self.views):
                    ctypes.memmove(ctypes.byref(plans[i]), ctypes.byref(pl), ctypes.sizeof(pl))
                    plans[i].row_start, plans[i].row_end = v.row_start, v.row_end
                    plans[i].block_rows = None
            else:
                kernels = [kernel_for(v, kname, order) for v in self.views]
                if len(set(kernels)) != 1:
                    kernels = ["staged"] * len(self.views)
                k = kernels[0]
                for i, v in enumerate(self.views):
                    pl = v.plan_for(k)
                    if pl is None:  # plan-free kernel: row range only
                        plans[i].row_start, plans[i].row_end = v.row_start, v.row_end
                    else:
                        ctypes.memmove(ctypes.byref(plans[i]), ctypes.byref(pl),
                                       ctypes.sizeof(pl))
            rec = (plans, _native.VARIANT_CODES[k])
            self._plans[key] = rec
        plans, code = rec
        dm = self.dm
        # no stream joins needed: x/y come from the host, and the previous
        # call returned only after its last copy (which waited for every
        # kernel) — the device buffers are free
        _native.check(_native.lib().dacsr_spmv_host_streamed(
            ctypes.byref(dm.desc), plans, len(self.views), code, int(order),
            x_host.ctypes.data, y_host.ctypes.data, self.x.data_ptr(), self.y.data_ptr(),
            float(alpha), float(beta), int(self.w), self.s_h2d.cuda_stream,
            self.s_comp.cuda_stream, self.s_d2h.cuda_stream, self.y_through_device),
            "dacsr_spmv_host_streamed")
        return y_host


def streamed(dm):
    sh = getattr(dm, "_streamed", None)
    if sh is None:
        sh = StreamedHost(dm)
        dm._streamed = sh
    return sh


__all__ = ["StreamedHost", "streamed"]
