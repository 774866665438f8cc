"""Device-resident matrices: HBM layout, row statistics and the row-block plan.

A ``DeviceMatrix`` owns the three arrays in HBM (torch tensors used only as
allocations), a ``dacsr_matrix_t`` descriptor for the C ABI, the row-length
statistics from ``dacsr_analyze`` and the nnz-balanced ROWBLOCK plan
(block table in HBM).  Layout rules:

* rowptr  int32 when nnz < 2^31, else int64 (C5 on one GPU); narrower host
  widths (int8/int16, reference test_spmv.py:238-247) widen to int32.
* inner   DA: int8/int16/int32 offsets kept as given (int16 is the paper's
  case, 2 bytes/entry); CSR: int32 (int64 only when ncols > 2^31).
* values  float32/float64 as given; ``astype`` makes float16/bfloat16
  copies (the width-lattice extension of model.py:21-74: 2-byte values,
  exact f32 products, f64 accumulation, one rounding on the store).
All arrays are unpadded and 16-byte aligned (torch allocations are 512-byte
aligned), which the TMA bulk copies require; kernels never read past nnz.

Host matrices cache their upload (they are immutable), so the reference-
style ``spmv(A, x, y)`` pays the operator transfer once.
"""

import ctypes

import numpy as np
import torch

from . import _native
from .core import CsrMatrix, DacsrMatrix

# kernels that run on the sliced layout (DeviceMatrix.build_slices)
SLICED_KERNELS = ("sliced", "sliced_pipe")
# kernels on a derived layout of the whole row range (any launch row range
# inside it): the sliced layout and the band-tiled layout
LAYOUT_KERNELS = SLICED_KERNELS + ("tiled",)

_KIND_NAME = {_native.KIND_CSR: "csr", _native.KIND_DA: "da"}


def _torch_device(device):
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.type != "cuda":
        raise ValueError(f"DeviceMatrix needs a CUDA device, got {device}")
    return device


def _upload(arr, dtype, device):
    a = np.ascontiguousarray(arr, dtype=dtype)
    if not a.flags.writeable:
        a = a.copy()
    return torch.from_numpy(a).to(device)


def _sync(stream=None):
    (stream if stream is not None else torch.cuda.current_stream()).synchronize()


def _stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class DeviceMatrix:
    """CSR or DA-CSR matrix in HBM plus its analysis and ROWBLOCK plan."""

    def __init__(self, kind, nrows, ncols, rowptr, colids, values, *, plan=True,
                 row_start=0, row_end=None, cap=None, long_len=None):
        if kind not in ("csr", "da"):
            raise ValueError(f"kind must be 'csr' or 'da', got {kind!r}")
        for t in (rowptr, colids, values):
            if not isinstance(t, torch.Tensor) or t.device.type != "cuda" or not t.is_contiguous():
                raise ValueError("rowptr/colids/values must be contiguous CUDA tensors")
        self.kind = kind
        self.nrows, self.ncols = int(nrows), int(ncols)
        self.rowptr, self.colids, self.values = rowptr, colids, values
        self.nnz = int(colids.numel())
        self.device = values.device
        self.desc = _native.Matrix(
            _native.KIND_DA if kind == "da" else _native.KIND_CSR,
            _native.dtype_code(rowptr.dtype), _native.dtype_code(colids.dtype),
            _native.dtype_code(values.dtype), self.nrows, self.ncols, self.nnz,
            rowptr.data_ptr(), colids.data_ptr() if self.nnz else None,
            values.data_ptr() if self.nnz else None)
        self.row_start = int(row_start)
        self.row_end = self.nrows if row_end is None else int(row_end)
        self.stats = None
        self.plan = None
        self._block_rows = None
        self._chunk_plans = {}
        self._sliced = None  # (plan, Slices, tensors) once build_slices ran
        self._tiled = None   # (plan, Tiles, tensors) once build_tiles ran
        self._launch_cache = {}
        self._spmv_fn = _native.lib().dacsr_spmv
        self._spmv_dev_alpha_fn = _native.lib().dacsr_spmv_dev_alpha
        self._spmv_dev_alpha_sumsq_fn = _native.lib().dacsr_spmv_dev_alpha_sumsq
        self.tuned_kernel = None
        if plan:
            self.build_plan(cap=cap, long_len=long_len)

    # ---- construction -------------------------------------------------
    @classmethod
    def from_host(cls, a, device=None, **kw):
        """Upload a host CsrMatrix/DacsrMatrix (widening narrow widths)."""
        device = _torch_device(device)
        if isinstance(a, DacsrMatrix):
            kind = "da"
            inner = a.colids.dtype if a.colids.dtype in (np.int8, np.int16, np.int32) else np.int32
        elif isinstance(a, CsrMatrix):
            kind = "csr"
            inner = np.int64 if a.ncols - 1 > np.iinfo(np.int32).max else np.int32
        else:
            raise TypeError(f"expected CsrMatrix or DacsrMatrix, got {type(a).__name__}")
        rp_dtype = np.int64 if a.nnz > np.iinfo(np.int32).max else np.int32
        with torch.cuda.device(device):
            rp = _upload(a.rowptr, rp_dtype, device)
            ci = _upload(a.colids, inner, device)
            va = _upload(a.values, a.values.dtype, device)
            return cls(kind, a.nrows, a.ncols, rp, ci, va, **kw)

    @classmethod
    def of(cls, a, device=None):
        """Cached device copy of an (immutable) host matrix."""
        if isinstance(a, DeviceMatrix):
            return a
        device = _torch_device(device)
        cache = a._device_cache()
        key = (device.type, device.index)
        dm = cache.get(key)
        if dm is None:
            dm = cls.from_host(a, device)
            cache[key] = dm
        return dm

    # ---- analysis and plan -------------------------------------------------
    def analyze(self, stream=None):
        st = _native.Stats()
        scratch = torch.empty(_native.ANALYZE_SCRATCH, dtype=torch.uint8, device=self.device)
        with torch.cuda.device(self.device):
            _native.check(_native.lib().dacsr_analyze(
                ctypes.byref(self.desc), self.row_start, self.row_end,
                ctypes.c_void_p(scratch.data_ptr()), ctypes.byref(st), _stream_ptr(stream)),
                "dacsr_analyze")
        self.stats = st
        return st

    def build_plan(self, cap=None, long_len=None, stream=None):
        L = _native.lib()
        st = self.stats or self.analyze(stream)
        if cap is None:
            cap = L.dacsr_plan_default_cap(ctypes.byref(st), self.desc.values_dtype,
                                           self.desc.colids_dtype)
        if long_len is None:
            long_len = int(max(128, 16 * np.ceil(max(st.mean_len, 1.0))))
        nb = L.dacsr_plan_nblocks(ctypes.byref(self.desc), st.entry_start, st.entry_end, cap)
        self._block_rows = torch.empty(nb + 1, dtype=torch.int64, device=self.device)
        plan = _native.Plan()
        with torch.cuda.device(self.device):
            _native.check(L.dacsr_plan_build(
                ctypes.byref(self.desc), self.row_start, self.row_end, st.entry_start,
                st.entry_end, int(cap), int(long_len),
                ctypes.c_void_p(self._block_rows.data_ptr()), ctypes.byref(plan),
                _stream_ptr(stream)), "dacsr_plan_build")
        self.plan = plan
        if hasattr(self, "_launch_cache"):
            self._launch_cache.clear()
        return plan

    def chunk_rows(self):
        """Rows per warp chunk.  32 (one per lane): measured faster than 64
        (two per lane) on C1/C2/C4 — the 64-row window halves the resident
        warps and serialises each lane's two rows (profiles/)."""
        return 32

    def chunk_window(self, rows=None, quantile=0.99):
        """Staging window (entries) for WSTREAM: the given quantile of the
        chunk entry counts plus the 16-byte alignment slack, rounded to 16."""
        rows = rows or self.chunk_rows()
        rs, re = self.row_start, self.row_end
        if re <= rs:
            return 64
        rp = self.rowptr[rs:re + 1].to(torch.int64)
        starts = rp[:-1:rows]
        ends = torch.cat([rp[rows::rows], rp[-1:]])[:starts.numel()]
        sizes = (ends - starts).to(torch.float64)
        q = float(torch.quantile(sizes, quantile).item()) if sizes.numel() > 1 else float(sizes.max())
        align = 16 // min(self.values.element_size(), self.colids.element_size())
        return int(min(16384, max(64, -(-(q + align) // 16) * 16)))

    def chunk_plan(self, vcap=None, rows=None, stream=None):
        """Plan copy carrying the WSTREAM chunk classification for a window
        of ``vcap`` entries over ``rows``-row chunks (defaults: planner's)."""
        rows = rows or self.chunk_rows()
        if vcap is None:
            vcap = self.chunk_window(rows)
        key = (vcap, rows)
        got = self._chunk_plans.get(key)
        if got is not None:
            return got[0]
        if self.plan is None:
            self.build_plan(stream=stream)
        plan = _native.Plan()
        ctypes.memmove(ctypes.byref(plan), ctypes.byref(self.plan), ctypes.sizeof(plan))
        nchunks = max(1, (self.row_end - self.row_start + rows - 1) // rows)
        chunks = torch.empty(nchunks, dtype=torch.int64, device=self.device)
        count = torch.empty(1, dtype=torch.int64, device=self.device)
        with torch.cuda.device(self.device):
            _native.check(_native.lib().dacsr_plan_chunks(
                ctypes.byref(self.desc), self.row_start, self.row_end, int(rows), int(vcap),
                ctypes.c_void_p(chunks.data_ptr()), ctypes.c_void_p(count.data_ptr()),
                ctypes.byref(plan), _stream_ptr(stream)), "dacsr_plan_chunks")
        plan.ctas_per_sm = getattr(self, "_ctas_per_sm", 0)
        self._chunk_plans[key] = (plan, chunks)
        self._launch_cache.clear()
        if None not in self._chunk_plans:
            self._chunk_plans[None] = self._chunk_plans[key]
        return plan

    # ---- sliced layout ------------------------------------------------------
    def slice_max_len(self, quantiles=(0.5, 0.75, 0.9, 0.95, 0.98, 0.99, 0.995, 0.999, 1.0)):
        """Longest row kept in the main slices: the candidate (a row-length
        quantile, <= 254) minimising an estimate of the work — 32 slots per
        unit of main-slice width, plus 2 per entry and 32 per row of the
        longer rows (medium slices / warp-per-row)."""
        rs, re = self.row_start, self.row_end
        if re <= rs:
            return 1
        lens = (self.rowptr[rs + 1:re + 1].to(torch.int64) - self.rowptr[rs:re].to(torch.int64))
        ns = (re - rs + 31) // 32
        padded = torch.zeros(ns * 32, dtype=torch.int64, device=self.device)
        padded[:re - rs] = lens
        padded = padded.view(ns, 32)
        qs = torch.quantile(lens.to(torch.float64)[:1 << 24],
                            torch.tensor(quantiles, dtype=torch.float64, device=self.device))
        cands = sorted({int(min(254, max(1, q))) for q in qs.ceil().tolist()})
        best, best_cost = cands[-1], None
        for t in cands:
            keep = torch.where(padded <= t, padded, torch.zeros_like(padded))
            out = padded > t
            cost = (32 * keep.max(dim=1).values.sum() + 2 * padded[out].sum()
                    + 32 * out.sum()).item()
            if best_cost is None or cost < best_cost:
                best, best_cost = t, cost
        return best

    def _scan(self, counts, out, sp):
        """out[0] = 0, out[k+1] = sum(counts[:k+1]) (int64, on the device)."""
        L = _native.lib()
        n = counts.numel()
        tb = ctypes.c_size_t(0)
        _native.check(L.dacsr_counts_to_rowptr(
            ctypes.c_void_p(counts.data_ptr()), n, ctypes.c_void_p(out.data_ptr()), _native.I64,
            None, ctypes.byref(tb), sp), "dacsr_counts_to_rowptr")
        tmp = torch.empty(max(int(tb.value), 1), dtype=torch.uint8, device=self.device)
        _native.check(L.dacsr_counts_to_rowptr(
            ctypes.c_void_p(counts.data_ptr()), n, ctypes.c_void_p(out.data_ptr()), _native.I64,
            ctypes.c_void_p(tmp.data_ptr()), ctypes.byref(tb), sp), "dacsr_counts_to_rowptr")

    def build_slices(self, max_len=None, medium_len=None, stream=None):
        """Build the sliced device layout (dacsr_slices_t) of rows
        [row_start, row_end): a bit-for-bit copy of the entries re-laid so a
        warp reads entry j of its 32 rows as one contiguous run.  Rows up to
        ``max_len`` entries sit in main slices, rows up to ``medium_len``
        (default max(max_len, 32)) in medium slices of 32 listed rows, longer
        rows are reduced warp by warp.  Returns the plan that carries it
        (variants "sliced" / "sliced_pipe")."""
        L = _native.lib()
        if self.plan is None:
            self.build_plan(stream=stream)
        if max_len is None:
            max_len = self.slice_max_len()
        max_len = int(min(254, max(1, max_len)))
        medium_len = int(min(254, max(max_len, 32 if medium_len is None else medium_len)))
        rs, re = self.row_start, self.row_end
        if re - rs >= 1 << 31:
            raise ValueError("the sliced layout addresses rows as int32 offsets (< 2^31 rows)")
        ns = (re - rs + 31) // 32
        dev = self.device
        sp = _stream_ptr(stream)
        vp = lambda t: ctypes.c_void_p(t.data_ptr())
        row_len = torch.zeros(max(re - rs, 1), dtype=torch.uint8, device=dev)
        counts = torch.zeros(3, max(ns, 1), dtype=torch.int32, device=dev)
        ptrs = torch.zeros(3, ns + 2, dtype=torch.int64, device=dev)
        with torch.cuda.device(dev):
            _native.check(L.dacsr_slices_count(
                ctypes.byref(self.desc), rs, re, max_len, medium_len, vp(row_len), vp(counts[0]),
                vp(counts[1]), vp(counts[2]), sp), "dacsr_slices_count")
            if ns:
                for k in range(3):
                    self._scan(counts[k, :ns], ptrs[k, :ns + 1], sp)
            total, n_medium, n_long = (int(v) for v in ptrs[:, ns].tolist())
            inner = torch.empty(max(total, 1), dtype=self.colids.dtype, device=dev)
            values = torch.empty(max(total, 1), dtype=self.values.dtype, device=dev)
            medium_rows = torch.empty(max(n_medium, 1), dtype=torch.int64, device=dev)
            long_rows = torch.empty(max(n_long, 1), dtype=torch.int64, device=dev)
            msl = (n_medium + 31) // 32
            m_ptr = torch.zeros(msl + 1, dtype=torch.int64, device=dev)
            sl = _native.Slices(rs, re, ns, total, max_len, medium_len, ptrs[0].data_ptr(),
                                row_len.data_ptr(), inner.data_ptr(), values.data_ptr(),
                                n_medium, msl, 0, medium_rows.data_ptr(), m_ptr.data_ptr(),
                                None, None, n_long, long_rows.data_ptr())
            _native.check(L.dacsr_slices_fill(ctypes.byref(self.desc), ctypes.byref(sl),
                                              vp(ptrs[1]), vp(ptrs[2]), sp), "dacsr_slices_fill")
            m_inner = m_values = None
            if n_medium:
                m_counts = torch.empty(msl, dtype=torch.int32, device=dev)
                _native.check(L.dacsr_slices_medium_count(ctypes.byref(sl), vp(m_counts), sp),
                              "dacsr_slices_medium_count")
                self._scan(m_counts, m_ptr, sp)
                m_total = int(m_ptr[-1].item())
                m_inner = torch.empty(max(m_total, 1), dtype=self.colids.dtype, device=dev)
                m_values = torch.empty(max(m_total, 1), dtype=self.values.dtype, device=dev)
                sl.m_total, sl.m_inner, sl.m_values = m_total, m_inner.data_ptr(), m_values.data_ptr()
                _native.check(L.dacsr_slices_medium_fill(ctypes.byref(self.desc), ctypes.byref(sl),
                                                         sp), "dacsr_slices_medium_fill")
            # the sliced kernels use programmatic dependent launch and read
            # the operator before griddepcontrol.wait: the layout must be
            # complete before any launch that follows
            _sync(stream)
        plan = _native.Plan()
        ctypes.memmove(ctypes.byref(plan), ctypes.byref(self.plan), ctypes.sizeof(plan))
        plan.slices = ctypes.addressof(sl)
        plan.tiles = self._tiled[0].tiles if self._tiled is not None else None
        plan.ctas_per_sm = getattr(self, "_ctas_per_sm", 0)
        tensors = {"row_len": row_len, "slice_ptr": ptrs[0], "inner": inner, "values": values,
                   "medium_rows": medium_rows, "m_slice_ptr": m_ptr, "m_inner": m_inner,
                   "m_values": m_values, "long_rows": long_rows}
        self._sliced = (plan, sl, tensors)
        self._invalidate_launches()
        return plan

    def build_tiles(self, tile_cols=None, stream=None):
        """Build the band-tiled device layout (dacsr_tiles_t) of rows
        [row_start, row_end) for the TILED kernel: 512-row groups, columns in
        tiles of ``tile_cols`` (default: the widest whose x ring fits the
        kernel's shared memory, dacsr_tiles_max_cols: 10416 for f64),
        each group's entries stored tile by tile in the order its lanes fold
        them.  A bit-for-bit copy of the entries (about the operator's size
        again in HBM, plus half a byte per row and tile of counts).  Returns
        the plan that carries it (variant "tiled")."""
        L = _native.lib()
        if self.plan is None:
            self.build_plan(stream=stream)
        widest = int(L.dacsr_tiles_max_cols(self.desc.values_dtype))
        if tile_cols is None:
            tile_cols = widest
        tile_cols = int(tile_cols)
        if tile_cols < 64 or tile_cols % 16 or tile_cols > widest:
            raise ValueError(f"tile_cols must be a multiple of 16 in [64, {widest}] (the x tiles "
                             "live in shared memory)")
        rs, re = self.row_start, self.row_end
        dev = self.device
        sp = _stream_ptr(stream)
        vp = lambda t: ctypes.c_void_p(t.data_ptr())
        ng = (re - rs + 511) // 512
        with torch.cuda.device(dev):
            ext = torch.empty(2, dtype=torch.int64, device=dev)
            _native.check(L.dacsr_tiles_extent(ctypes.byref(self.desc), rs, re, vp(ext), sp),
                          "dacsr_tiles_extent")
            cmin, cmax = (int(v) for v in ext.tolist())
            if cmax < cmin:  # no entries
                cmin = cmax = 0
            tile_lo = torch.zeros(max(ng, 1), dtype=torch.int32, device=dev)
            skip = torch.zeros(max(32 * ng, 1), dtype=torch.int16, device=dev)  # uint16 bits
            tl = _native.Tiles(rs, re, ng, cmin, cmax, tile_cols, L.dacsr_tiles_step_group(), 0, 0,
                               None, None,
                               tile_lo.data_ptr(), None, skip.data_ptr(), None, None, 0, None,
                               None, None)
            cnt = torch.zeros(3, max(ng, 1), dtype=torch.int32, device=dev)
            _native.check(L.dacsr_tiles_count(ctypes.byref(self.desc), ctypes.byref(tl),
                                               vp(cnt[0]), vp(cnt[1]), vp(cnt[2]), sp),
                          "dacsr_tiles_count")
            ptrs = torch.zeros(3, ng + 1, dtype=torch.int64, device=dev)
            if ng:
                for k in range(3):
                    self._scan(cnt[k, :ng], ptrs[k, :ng + 1], sp)
            nblocks, total, n_ovf = (int(v) for v in ptrs[:, ng].tolist())
            counts = torch.empty(max(32 * nblocks, 1), dtype=torch.int64, device=dev)  # uint64 bits
            masks = torch.empty(max(nblocks, 1), dtype=torch.int64, device=dev)  # uint64 bits
            order = torch.empty(max(32 * nblocks, 1), dtype=torch.int64, device=dev)  # uint64 bits
            inner = torch.zeros(total + 16, dtype=self.colids.dtype, device=dev)
            values = torch.zeros(total + 16, dtype=self.values.dtype, device=dev)
            ovf_rows = torch.empty(max(n_ovf, 1), dtype=torch.int64, device=dev)
            tl.total, tl.nblocks, tl.n_ovf = total, nblocks, n_ovf
            tl.cnt_ptr, tl.ent_ptr = ptrs[0].data_ptr(), ptrs[1].data_ptr()
            tl.counts, tl.inner, tl.values = counts.data_ptr(), inner.data_ptr(), values.data_ptr()
            tl.ovf_rows, tl.masks, tl.order = ovf_rows.data_ptr(), masks.data_ptr(), order.data_ptr()
            _native.check(L.dacsr_tiles_fill(ctypes.byref(self.desc), ctypes.byref(tl),
                                              vp(ptrs[2]), sp), "dacsr_tiles_fill")
            _sync(stream)
        plan = _native.Plan()
        ctypes.memmove(ctypes.byref(plan), ctypes.byref(self.plan), ctypes.sizeof(plan))
        plan.slices = self._sliced[0].slices if self._sliced is not None else None
        plan.tiles = ctypes.addressof(tl)
        tensors = {"ptrs": ptrs, "tile_lo": tile_lo, "skip": skip, "counts": counts,
                   "masks": masks, "order": order, "inner": inner, "values": values, "ovf_rows": ovf_rows}
        self._tiled = (plan, tl, tensors)
        self._invalidate_launches()
        return plan

    def tiles_info(self):
        """Summary of the band-tiled layout (None before build_tiles)."""
        if self._tiled is None:
            return None
        _, tl, tensors = self._tiled
        ng = max(1, tl.ngroups)
        return {"tile_cols": tl.tile_cols, "step_group": tl.step_group, "col0": tl.col0,
                "cmax": tl.cmax,
                "groups": tl.ngroups, "tile_blocks": tl.nblocks,
                "tiles_per_group": tl.nblocks / ng, "entries": tl.total, "n_ovf": tl.n_ovf,
                "count_bytes_per_row": (16 * 32 + 8) * tl.nblocks / max(1, tl.row_end - tl.row_start),
                "bytes": sum(t.numel() * t.element_size() for t in tensors.values())}

    def _invalidate_launches(self):
        """Forget cached launch records and host-path plans (they hold raw
        pointers into the layouts)."""
        self._launch_cache.clear()
        if getattr(self, "_streamed", None) is not None:
            self._streamed._plans.clear()

    def slices_info(self):
        """Summary of the sliced layout (None before build_slices)."""
        if self._sliced is None:
            return None
        _, sl, tensors = self._sliced
        return {"max_len": sl.max_len, "medium_len": sl.medium_len, "slots": sl.total,
                "n_medium": sl.n_medium, "m_slots": sl.m_total, "n_long": sl.n_long,
                "nslices": sl.nslices,
                "padding": (sl.total + sl.m_total) / max(1, self.nnz) - 1.0,
                "bytes": sum(t.numel() * t.element_size() for t in tensors.values()
                             if t is not None)}

    def autotune(self, candidates=("tiled", "sliced_pipe", "sliced", "wstream", "scalar",
                                   "rowblock"),
                 cold=False, x=None, reps=5, tune_layout=True):
        """Time the exact naive-order kernels on this matrix and remember the
        fastest for variant "naive"/"auto" (all give bit-identical results,
        so this only changes speed; without autotune the row-statistics
        selection of dacsr_select_variant applies).  With ``tune_layout``
        the sliced layout's width (max_len) and its L2-prefetch flag are
        chosen too; otherwise the current layout is kept.  Derived layouts
        of kernels that lose are released.  Returns {kernel: seconds}."""
        from .harness import time_kernel
        if x is None:
            x = torch.ones(self.ncols, dtype=self.values.dtype, device=self.device)
        y = torch.empty(self.nrows, dtype=self.values.dtype, device=self.device)
        times = {}

        def timed(k):
            fn = lambda: self.spmv_into(x, y, 1.0, 0.0, k, 0)
            return time_kernel(fn, epochs=3, warmup_iters=2, min_epoch_iters=reps,
                               min_epoch_time=0.0, cold=cold, graph=0 if cold else reps)

        sliced = [k for k in candidates if k in SLICED_KERNELS]
        flag = True
        if tune_layout and sliced and self.plan is not None and self.nnz:
            # the main/medium split changes the slice widths a warp walks:
            # time the cost model's choice against 8 and 16 (one batch or
            # two per slice), each with and without the L2 prefetch, and keep
            # the fastest (layout, flag)
            model = self.slice_max_len()
            longest = int(self.stats.max_len) if self.stats is not None else 254
            probe = "sliced_pipe" if "sliced_pipe" in sliced else sliced[0]
            tried = {}
            for t in sorted({min(v, max(1, longest)) for v in (model, 8, 16)}):
                self.build_slices(t)
                for on in (True, False):
                    self.set_sliced_l2_prefetch(on)
                    tried[(t, on)] = timed(probe)
            (best_t, flag), _ = min(tried.items(), key=lambda kv: kv[1])
            if self._sliced[1].max_len != best_t:
                self.build_slices(best_t)
            self.slice_max_len_tuned = {f"{k[0]}{'' if k[1] else ':no_l2_prefetch'}": v
                                        for k, v in tried.items()}
        if self._sliced is not None:
            self.set_sliced_l2_prefetch(flag)
        flags = {}
        for k in candidates:
            if k in ("wstream", "rowblock", "tiled") + SLICED_KERNELS and self.plan is None:
                continue
            if k in SLICED_KERNELS and tune_layout and self.nnz:
                # the prefetch flag was chosen on the probe kernel; the other
                # sliced kernel may want the opposite (SLICED has no offset
                # pipeline and leans on the prefetch), so each is timed both ways
                both = {}
                for on in (flag, not flag):
                    self.set_sliced_l2_prefetch(on)
                    both[on] = timed(k)
                flags[k] = min(both, key=both.get)
                times[k] = both[flags[k]]
            else:
                times[k] = timed(k)
        best = min(times, key=times.get)
        self.tuned_kernel = best
        if best in flags:
            self.set_sliced_l2_prefetch(flags[best])
        if best not in SLICED_KERNELS and self._sliced is not None:
            self._sliced = None  # the sliced copy of the entries was only built to be timed
        if best != "tiled" and self._tiled is not None:
            self._tiled = None
        self._invalidate_launches()
        return times

    def set_sliced_l2_prefetch(self, on):
        """Enable / disable the sliced kernels' L2 bulk prefetch of the slice
        two steps ahead (dacsr_plan_t.flags)."""
        if self._sliced is None:
            return
        plan = self._sliced[0]
        if on:
            plan.flags &= ~_native.PLAN_NO_L2_PREFETCH
        else:
            plan.flags |= _native.PLAN_NO_L2_PREFETCH
        self._invalidate_launches()

    def set_ctas_per_sm(self, n):
        """Cap WSTREAM's resident CTAs per SM (0 = occupancy maximum)."""
        for plan, _ in self._chunk_plans.values():
            plan.ctas_per_sm = int(n)
        if self._sliced is not None:
            self._sliced[0].ctas_per_sm = int(n)
        self._ctas_per_sm = int(n)
        self._invalidate_launches()

    def set_chunk_window(self, vcap, rows=None):
        """Pin the WSTREAM staging window (entries, multiple of 16) and the
        rows per warp chunk (32 or 64)."""
        rows = rows or self.chunk_rows()
        self.chunk_plan(int(vcap), rows)
        self._chunk_plans[None] = self._chunk_plans[(int(vcap), rows)]
        self._launch_cache.clear()

    def plan_for(self, kname, row_start=None, row_end=None):
        """The plan a kernel needs (None when it needs none or the row range
        differs from the planned one)."""
        rs = self.row_start if row_start is None else row_start
        re = self.row_end if row_end is None else row_end
        if kname in SLICED_KERNELS:  # any row range inside theirs
            if not (self.row_start <= rs <= re <= self.row_end):
                return None
            return self._sliced[0] if self._sliced is not None else self.build_slices()
        if kname == "tiled":
            if not (self.row_start <= rs <= re <= self.row_end):
                return None
            return self._tiled[0] if self._tiled is not None else self.build_tiles()
        if self.plan is None or rs != self.plan.row_start or re != self.plan.row_end:
            return None
        if kname == "wstream":
            got = self._chunk_plans.get(None)
            return got[0] if got is not None else self.chunk_plan()
        return self.plan

    # ---- properties -----------------------------------------------------------
    @property
    def iindex_width(self):
        return self.colids.element_size() * 8

    @property
    def oindex_width(self):
        return self.rowptr.element_size() * 8

    @property
    def scalar_width(self):
        return self.values.element_size() * 8

    @property
    def dtype(self):
        return self.values.dtype

    def astype(self, dtype, plan=True):
        """The same operator with values converted on the device (torch's
        rounding) to ``dtype`` (float16/bfloat16/float32/float64); rowptr and
        offsets are shared.  x and y must then carry the same dtype."""
        dtype = getattr(torch, dtype) if isinstance(dtype, str) else dtype
        if dtype not in (torch.float16, torch.bfloat16, torch.float32, torch.float64):
            raise ValueError(f"unsupported value dtype {dtype}")
        if dtype == self.values.dtype:
            return self
        return DeviceMatrix(self.kind, self.nrows, self.ncols, self.rowptr, self.colids,
                            self.values.to(dtype), plan=plan, row_start=self.row_start,
                            row_end=self.row_end)

    def storage_bytes(self):
        return sum(t.numel() * t.element_size() for t in (self.rowptr, self.colids, self.values))

    # ---- the multiply ---------------------------------------------------------
    def spmv_into(self, x, y, alpha=1.0, beta=0.0, variant="rowblock", order=0, x_offset=0,
                  row_start=None, row_end=None, stream=None, group_sumsq=None):
        """Launch y = alpha*A@x + beta*y on device tensors (no validation
        beyond the C ABI's; ``spmv`` is the validating entry point).
        ``alpha`` may be a one-element float64 CUDA tensor: the kernel reads it
        from device memory (dacsr_spmv_dev_alpha; no alpha == 0 short-cut).
        ``group_sumsq`` (with a device alpha, TILED only; see
        ``fused_sumsq_ok``): a float64 tensor that receives the sum of y^2 of
        every 512-row group at index row // 512 (dacsr_spmv_dev_alpha_sumsq).

        The (variant, order, row range) -> (code, plan) resolution is cached
        per matrix, so a launch costs one ctypes call (a few microseconds of
        host time — it sits between back-to-back kernels)."""
        key = (variant, order, row_start, row_end)
        rec = self._launch_cache.get(key)
        if rec is None:
            code = _native.VARIANT_CODES[variant] if isinstance(variant, str) else int(variant)
            rs = self.row_start if row_start is None else int(row_start)
            re = self.row_end if row_end is None else int(row_end)
            plan = self.plan_for(variant if isinstance(variant, str) else "", rs, re)
            rec = (ctypes.byref(self.desc), ctypes.byref(plan) if plan is not None else None,
                   code, int(order), rs, re, plan)
            self._launch_cache[key] = rec
        desc, plan_ref, code, order_code, rs, re, _ = rec
        if stream is None:
            sp = torch.cuda.current_stream(self.device).cuda_stream
        else:
            sp = stream.cuda_stream
        if group_sumsq is not None:
            if not isinstance(alpha, torch.Tensor):
                raise TypeError("group_sumsq needs alpha as a one-element float64 CUDA tensor "
                                "(dacsr_spmv_dev_alpha_sumsq reads it on the device)")
            status = self._spmv_dev_alpha_sumsq_fn(desc, plan_ref, code, order_code,
                                                   x.data_ptr() if x is not None else None,
                                                   x_offset, y.data_ptr(), alpha.data_ptr(), beta,
                                                   rs, re, group_sumsq.data_ptr(), sp)
        elif isinstance(alpha, torch.Tensor):  # alpha in device memory (one float64)
            status = self._spmv_dev_alpha_fn(desc, plan_ref, code, order_code,
                                             x.data_ptr() if x is not None else None, x_offset,
                                             y.data_ptr(), alpha.data_ptr(), beta, rs, re, sp)
        else:
            status = self._spmv_fn(desc, plan_ref, code, order_code,
                                   x.data_ptr() if x is not None else None, x_offset,
                                   y.data_ptr(), alpha, beta, rs, re, sp)
        if status:
            _native.check(status, "dacsr_spmv")
        return y

    def fused_sumsq_ok(self, variant, order=0, row_start=None, row_end=None):
        """True if spmv_into(..., group_sumsq=...) can run for this variant
        and row range: the TILED kernel in the naive order, its layout built
        from a row that is a multiple of 512 with no rows left out, and the
        range made of whole 512-row groups (dacsr_spmv_dev_alpha_sumsq)."""
        if variant != "tiled" or order != _native.ORDER_NAIVE:
            return False
        if self._tiled is None:
            self.build_tiles()
        tl = self._tiled[1]
        rs = self.row_start if row_start is None else int(row_start)
        re = self.row_end if row_end is None else int(row_end)
        return (tl.n_ovf == 0 and tl.row_start % 512 == 0 and (rs - tl.row_start) % 512 == 0
                and (re == tl.row_end or (re - tl.row_start) % 512 == 0))

    def __repr__(self):
        return (f"DeviceMatrix({self.kind}, {self.nrows}x{self.ncols}, nnz={self.nnz}, "
                f"rowptr={self.rowptr.dtype}, inner={self.colids.dtype}, "
                f"values={self.values.dtype}, device={self.device})")


def bandwidth_device(dm, stream=None):
    """max |col - row| of a DeviceMatrix, computed in HBM."""
    out = torch.zeros(1, dtype=torch.int64, device=dm.device)
    with torch.cuda.device(dm.device):
        _native.check(_native.lib().dacsr_bandwidth(ctypes.byref(dm.desc),
                                                    ctypes.c_void_p(out.data_ptr()),
                                                    _stream_ptr(stream)), "dacsr_bandwidth")
    return int(out.item())


def to_dacsr_device(dm, iindex=16, stream=None):
    """Device-side CSR → DA-CSR (reference core.py:334-355) with the same
    int-k fit check; rowptr and values are shared, offsets are new."""
    from .core import index_max
    from .errors import BandwidthExceedsIndexRange
    if dm.kind != "csr":
        raise TypeError("to_dacsr_device expects a CSR DeviceMatrix")
    limit = index_max(iindex)
    w = bandwidth_device(dm, stream)
    if w > limit:
        raise BandwidthExceedsIndexRange(
            f"bandwidth {w} exceeds the {iindex}-bit signed offset range [-{limit}, {limit}]")
    tdt = {8: torch.int8, 16: torch.int16, 32: torch.int32}[iindex]
    off = torch.empty(dm.nnz, dtype=tdt, device=dm.device)
    with torch.cuda.device(dm.device):
        _native.check(_native.lib().dacsr_csr_to_da(
            ctypes.byref(dm.desc), ctypes.c_void_p(off.data_ptr()), _native.dtype_code(tdt),
            _stream_ptr(stream)), "dacsr_csr_to_da")
    return DeviceMatrix("da", dm.nrows, dm.ncols, dm.rowptr, off, dm.values,
                        row_start=dm.row_start, row_end=dm.row_end)


__all__ = ["DeviceMatrix", "bandwidth_device", "to_dacsr_device"]
