"""The SpMV operator API: ``y <- alpha*A@x + beta*y`` on the B200.

Mirrors the reference operator (/root/reference/pkg/src/dacsr/spmv/
__init__.py:104-183) argument for argument and error for error:

* ``a``: CsrMatrix | DacsrMatrix (host, uploaded once and cached) or a
  ``DeviceMatrix``; anything else → TypeError                    (117-122)
* ``x`` shape (ncols,) else DimensionMismatch                      (123-127)
* ``y=None`` allowed only when beta == 0 (fresh output) else ValueError;
  ``y`` updated in place and returned (the same object)           (130-140)
* values/x/y share float32|float64 else UnsupportedScalarWidth     (141-146)
* alpha == 0: the matrix and x are not touched; y = 0 (beta == 0),
  y *= beta (beta ∉ {0, 1}), unchanged (beta == 1)                (150-156)
* beta == 0: y is never read (NaN-safe)
* ``variant``: the reference names run their exact summation order on the
  GPU, bit-identical to the reference kernels; ``ParallelRowBlock(T, inner)``
  is bit-identical to ``inner`` (reference guarantee) and runs as one launch.
  GPU-specific names: "auto", "rowblock", "staged", "scalar", "vector2",
  "vector4", "vector8", "vector16", "warp" (the vector/warp variants and
  "rowblock_tree" combine lanes by a tree: within 2^-40, not bit-exact).
* ``backend``: only None / "cuda" — there is one backend and no fallback.

Host numpy x/y are copied to/from the device inside the call (pinned host
memory gives async DMA); torch CUDA tensors stay on the device.
"""

import contextlib
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .core import CsrMatrix, DacsrMatrix
from .device import DeviceMatrix, _stream_ptr
from .errors import DimensionMismatch, UnsupportedScalarWidth

ENV_FLAG = "DACSR_BACKEND"
STREAMED_MIN_ROWS = 1 << 18  # host-array calls at least this tall use the streamed path

SERIAL_VARIANTS = ("naive", "shifted_base", "multi_accumulator_3", "strip_mined_4")

# reference variant -> (kernel variant, summation order); "exact" is resolved
# per matrix by the library's selection policy (dacsr_select_variant)
_EXACT = {
    "naive": ("exact", _native.ORDER_NAIVE),
    "shifted_base": ("exact", _native.ORDER_NAIVE),
    "multi_accumulator_3": ("exact", _native.ORDER_MACC3),
    "strip_mined_4": ("exact", _native.ORDER_STRIP4),
}
_EXACT_KERNELS = ("rowblock", "staged", "scalar", "wstream", "sliced", "sliced_pipe", "tiled")
_SLICED = ("sliced", "sliced_pipe")  # the sliced layout
_TREE_KERNELS = ("vector2", "vector4", "vector8", "vector16", "warp")
GPU_VARIANTS = ("auto", "rowblock_tree") + _EXACT_KERNELS + _TREE_KERNELS
_CODE_NAME = {v: k for k, v in _native.VARIANT_CODES.items()}


def available_backends():
    """Backends usable in this process: the CUDA library only."""
    return ("cuda",)


def default_backend():
    """Backend named by DACSR_BACKEND (auto/cuda); anything else is rejected."""
    choice = os.environ.get(ENV_FLAG, "auto")
    if choice not in ("auto", "cuda"):
        raise ValueError(f"{ENV_FLAG} must be auto or cuda, got {choice!r}")
    return "cuda"


@dataclass(frozen=True)
class ParallelRowBlock:
    """Row-block parallel form of a serial variant (reference 55-68).

    On the GPU every launch is already row-parallel; the result is
    bit-identical to ``inner`` exactly as the reference guarantees.
    """

    threads: int
    inner: str = "naive"

    def __post_init__(self):
        if not isinstance(self.threads, (int, np.integer)) or self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.inner not in SERIAL_VARIANTS:
            raise ValueError(f"inner variant must be one of {SERIAL_VARIANTS}, got {self.inner!r}")


def row_blocks(rowptr, nblocks):
    """``nblocks`` contiguous nnz-balanced row ranges covering [0, nrows)
    (reference 71-85: cut k at searchsorted(rowptr, k*nnz//nblocks, 'left'),
    clamped monotone).  Used by the multi-GPU row partition."""
    rp = np.asarray(rowptr)
    nrows = len(rp) - 1
    nnz = int(rp[-1])
    cuts = [0]
    for k in range(1, nblocks):
        b = int(np.searchsorted(rp, (k * nnz) // nblocks, side="left"))
        cuts.append(min(max(b, cuts[-1]), nrows))
    cuts.append(nrows)
    return list(zip(cuts[:-1], cuts[1:]))


def resolve_variant(variant):
    """(kernel variant name, order code) for a user-facing variant."""
    if isinstance(variant, ParallelRowBlock):
        variant = variant.inner
    if isinstance(variant, str):
        if variant in _EXACT:
            return _EXACT[variant]
        if variant == "rowblock_tree":
            return "rowblock", _native.ORDER_TREE
        if variant == "auto":
            return "exact", _native.ORDER_NAIVE
        if variant in _EXACT_KERNELS:
            return variant, _native.ORDER_NAIVE
        if variant in _TREE_KERNELS:
            return variant, _native.ORDER_TREE
    raise ValueError(
        f"unknown variant {variant!r}; expected one of {SERIAL_VARIANTS + GPU_VARIANTS} "
        "or a ParallelRowBlock")


# rows the tiled layout may leave to its warp-per-row pass before the
# selection falls back (rows with more than 15 entries inside one column
# tile: dense rows in a narrow band)
TILED_MAX_LEFT_OUT = 0.01


def _tiled_layout_fits(dm):
    """The selection picked TILED from the gather scatter; build its layout
    (needed anyway) and keep it only if nearly every row is in it."""
    ok = getattr(dm, "_tiled_fits", None)
    if ok is None:
        dm.plan_for("tiled")
        info = dm.tiles_info()
        ok = info["n_ovf"] <= TILED_MAX_LEFT_OUT * max(1, dm.row_end - dm.row_start)
        if not ok:
            dm._tiled = None  # release the layout
            dm._invalidate_launches()
        dm._tiled_fits = ok
    return ok


def kernel_for(dm, kname, order):
    """Concrete kernel name for a resolved (name, order) on this matrix."""
    if kname == "exact":
        if order == _native.ORDER_NAIVE and getattr(dm, "tuned_kernel", None):
            return dm.tuned_kernel      # DeviceMatrix.autotune() picked it
        if dm.stats is None:
            return "staged"
        kname = _CODE_NAME[_native.lib().dacsr_select_variant(dm.stats, order)]
        if kname == "tiled" and dm.plan is not None and not _tiled_layout_fits(dm):
            kname = "sliced_pipe"
        if (kname == "sliced_pipe" and dm.values.element_size() == 2
                and dm.stats.max_len <= 64 and dm.stats.cv_len <= 0.5):
            # 16-bit values (the f16 / bf16 extension) on regular rows: the
            # sliced kernels are issue-bound there and thread-per-row from the
            # CSR arrays is faster (C2-bf16: 17 against 21 us warm, 27 against
            # 33 cold); the C ABI's selection does not see the value type
            kname = "scalar"
    if kname in ("wstream", "tiled") + _SLICED and order in (_native.ORDER_MACC3,
                                                             _native.ORDER_STRIP4):
        kname = "rowblock"  # warp streams / slices / tiles specialise the naive order
    if kname in ("rowblock", "wstream", "tiled") + _SLICED and dm.plan is None:
        return "staged"
    return kname


_SCALARS = ("float32", "float64")
_SCALARS_16 = ("float16", "bfloat16")  # DeviceMatrix.astype extension only


def _is_host(v):
    return isinstance(v, np.ndarray)


def _as_vector(v, name):
    if isinstance(v, torch.Tensor):
        return v
    return np.asarray(v)


def _dtype_name(v):
    return str(v.dtype).replace("torch.", "")


def _to_device(v, device):
    """Host numpy → device tensor (async DMA when v is in pinned memory)."""
    t = torch.from_numpy(np.ascontiguousarray(v) if v.flags.writeable
                         else np.array(v, copy=True))
    return t.to(device, non_blocking=t.is_pinned())


def spmv(a, x, y=None, alpha=1.0, beta=0.0, variant="naive", backend=None, *, stream=None):
    """Compute ``y <- alpha*A@x + beta*y`` on the GPU and return ``y``."""
    if isinstance(a, (CsrMatrix, DacsrMatrix)):
        nrows, ncols, vdtype = a.nrows, a.ncols, str(a.values.dtype)
    elif isinstance(a, DeviceMatrix):
        nrows, ncols, vdtype = a.nrows, a.ncols, _dtype_name(a.values)
    else:
        raise TypeError(f"expected CsrMatrix or DacsrMatrix, got {type(a).__name__}")
    x = _as_vector(x, "x")
    if tuple(x.shape) != (ncols,):
        raise DimensionMismatch(f"x has shape {tuple(x.shape)}, expected ({ncols},)")
    alpha = float(alpha)
    beta = float(beta)
    fresh = y is None
    if fresh:
        if beta != 0.0:
            raise ValueError("y must be provided when beta != 0")
    else:
        if not isinstance(y, (np.ndarray, torch.Tensor)):
            raise TypeError("y must be a numpy array or torch tensor (it is updated in place)")
        if tuple(y.shape) != (nrows,):
            raise DimensionMismatch(f"y has shape {tuple(y.shape)}, expected ({nrows},)")
    if vdtype not in _SCALARS and not (isinstance(a, DeviceMatrix) and vdtype in _SCALARS_16):
        raise UnsupportedScalarWidth(f"unsupported scalar dtype {vdtype}")
    ydtype = vdtype if fresh else _dtype_name(y)
    if _dtype_name(x) != vdtype or ydtype != vdtype:
        raise UnsupportedScalarWidth(
            f"scalar widths disagree: matrix {vdtype}, x {_dtype_name(x)}, y {ydtype}")
    if backend is None:
        default_backend()
    elif backend != "cuda":
        raise ValueError(f"unknown backend {backend!r}; only 'cuda' is available")
    kname, order = resolve_variant(variant)  # validate before touching anything

    if fresh:
        y = (np.empty(nrows, dtype=vdtype) if _is_host(x) else
             torch.empty(nrows, dtype=x.dtype, device=x.device))

    dm = DeviceMatrix.of(a, None if not isinstance(x, torch.Tensor) else x.device)
    kname = kernel_for(dm, kname, order)
    dev = dm.device
    if isinstance(y, torch.Tensor) and y.device != dev:
        raise ValueError(f"y is on {y.device}, matrix on {dev}")
    if isinstance(x, torch.Tensor) and x.device != dev:
        raise ValueError(f"x is on {x.device}, matrix on {dev}")
    if isinstance(y, torch.Tensor) and not y.is_contiguous():
        raise ValueError("y must be contiguous")

    # a caller-supplied stream becomes the current stream for the whole call:
    # host->device copies, the kernel and the device->host copy are then
    # ordered on it (and temporaries are allocated on it)
    stream_ctx = torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
    with torch.cuda.device(dev), stream_ctx:
        y_dev = y if isinstance(y, torch.Tensor) else None
        if alpha == 0.0:
            # matrix and x untouched (reference 150-156); y = beta*y on device
            if beta == 1.0 or nrows == 0:
                return y
            if y_dev is None:
                y_dev = (torch.empty(nrows, dtype=dm.values.dtype, device=dev) if beta == 0.0
                         else _to_device(y, dev))
            _native.check(_native.lib().dacsr_scale(
                _native.ctypes.c_void_p(y_dev.data_ptr()), _native.dtype_code(dm.values.dtype),
                nrows, beta, _stream_ptr(None)), "dacsr_scale")
        elif (not isinstance(x, torch.Tensor) and not isinstance(y, torch.Tensor)
              and nrows >= STREAMED_MIN_ROWS and dm.nnz and stream is None):
            # host in, host out: x streams in by row pieces while earlier
            # pieces compute and their y streams back (hostpath.py)
            from .hostpath import streamed
            y_host = y if y.flags.c_contiguous and y.flags.writeable else None
            if y_host is None:
                raise ValueError("y must be a writable C-contiguous array")
            return streamed(dm).run(np.ascontiguousarray(x), y_host, alpha, beta, kname, order)
        else:
            x_dev = x.contiguous() if isinstance(x, torch.Tensor) else _to_device(x, dev)
            if y_dev is None:
                y_dev = (torch.empty(nrows, dtype=dm.values.dtype, device=dev) if beta == 0.0
                         else _to_device(y, dev))
            if nrows:
                dm.spmv_into(x_dev if ncols else None, y_dev, alpha, beta, kname, order)
        if not isinstance(y, torch.Tensor) and nrows:
            out = torch.from_numpy(y)
            out.copy_(y_dev, non_blocking=out.is_pinned())
            if out.is_pinned():
                torch.cuda.current_stream().synchronize()
    return y


def work_flops(a=None, *, nnz=None, nrows=None):
    """Floating-point work of one SpMV: 2*nnz + 2*nrows (reference 186-193)."""
    if a is not None:
        nnz, nrows = a.nnz, a.nrows
    return 2 * nnz + 2 * nrows


__all__ = ["ENV_FLAG", "GPU_VARIANTS", "ParallelRowBlock", "SERIAL_VARIANTS",
           "available_backends", "default_backend", "resolve_variant", "row_blocks", "spmv",
           "work_flops"]
