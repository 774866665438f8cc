"""Device-side generation of the random banded configurations (C3, C5).

Thin host wrapper over ``dacsr_gen_banded_counts`` / ``_fill`` /
``dacsr_counts_to_rowptr`` (csrc/gen.cu).  The matrix never exists on the
host: at C5 it is 2.1e9 entries.  Any row range [r0, r1) can be produced on
its own (a rank's block), identical to the same rows of the whole matrix.
The CPU checker is oracle/gen_oracle.c (tests only).
"""

import ctypes

import numpy as np
import torch

from . import _native
from .device import DeviceMatrix, _stream_ptr
from .workloads import BANDED_CONFIGS, normal_table, poisson_cdf

_I32_MAX = np.iinfo(np.int32).max


def _vp(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def tables(lam, kmax, device):
    cdf = torch.from_numpy(poisson_cdf(lam, kmax)).to(device)
    table = torch.from_numpy(normal_table()).to(device)
    return cdf, table


def banded_arrays(n, b, lam, kmax, seed, device, r0=0, r1=None, kinds=("da",),
                  values_dtype=torch.float64, stream=None):
    """Rows [r0, r1) as device tensors: dict with rowptr (local, from 0),
    offsets (int16, if "da" in kinds), colids (int32 absolute, if "csr"),
    values."""
    r1 = n if r1 is None else r1
    L = _native.lib()
    sp = _stream_ptr(stream)
    cdf, table = tables(lam, kmax, device)
    m = r1 - r0
    counts = torch.empty(max(m, 1), dtype=torch.int32, device=device)
    _native.check(L.dacsr_gen_banded_counts(n, b, kmax, seed, _vp(cdf), r0, r1, _vp(counts), sp),
                  "dacsr_gen_banded_counts")
    rowptr = torch.empty(m + 1, dtype=torch.int64, device=device)
    tmp_bytes = ctypes.c_size_t(0)
    _native.check(L.dacsr_counts_to_rowptr(_vp(counts), m, _vp(rowptr), _native.I64, None,
                                           ctypes.byref(tmp_bytes), sp), "counts_to_rowptr")
    tmp = torch.empty(max(tmp_bytes.value, 1), dtype=torch.uint8, device=device)
    _native.check(L.dacsr_counts_to_rowptr(_vp(counts), m, _vp(rowptr), _native.I64, _vp(tmp),
                                           ctypes.byref(tmp_bytes), sp), "counts_to_rowptr")
    del counts, tmp
    nnz = int(rowptr[-1].item())
    if nnz <= _I32_MAX:
        rowptr = rowptr.to(torch.int32)
    out = {"rowptr": rowptr, "nnz": nnz}
    offsets = torch.empty(nnz, dtype=torch.int16, device=device) if "da" in kinds else None
    colids = torch.empty(nnz, dtype=torch.int32, device=device) if "csr" in kinds else None
    values = torch.empty(nnz, dtype=values_dtype, device=device)
    _native.check(L.dacsr_gen_banded_fill(
        n, b, kmax, seed, _vp(cdf), _vp(table), r0, r1, _vp(rowptr),
        _native.dtype_code(rowptr.dtype), _vp(offsets), _vp(colids), _vp(values),
        _native.dtype_code(values_dtype), sp), "dacsr_gen_banded_fill")
    out.update(offsets=offsets, colids=colids, values=values)
    return out


def banded_device(config, device=None, kinds=("da", "csr"), values_dtype=torch.float64,
                  r0=0, r1=None, plan=True):
    """DeviceMatrix objects for config "c3"/"c5" (or an explicit tuple
    (n, b, lam, kmax, seed)); returns {kind: DeviceMatrix} sharing values."""
    n, b, lam, kmax, seed = BANDED_CONFIGS[config] if isinstance(config, str) else config
    device = torch.device(device or "cuda")
    r1 = n if r1 is None else r1
    arr = banded_arrays(n, b, lam, kmax, seed, device, r0, r1, kinds, values_dtype)
    out = {}
    if "da" in kinds:
        out["da"] = DeviceMatrix("da", r1 - r0, n, arr["rowptr"], arr["offsets"], arr["values"],
                                 plan=plan)
    if "csr" in kinds:
        out["csr"] = DeviceMatrix("csr", r1 - r0, n, arr["rowptr"], arr["colids"], arr["values"],
                                  plan=plan)
    return out


def normal_vector(n, seed, device, dtype=torch.float64, i0=0):
    """x[i] = N(H(seed, i0 + i)) on the device (same quantile transform)."""
    table = torch.from_numpy(normal_table()).to(device)
    out = torch.empty(n, dtype=dtype, device=device)
    _native.check(_native.lib().dacsr_gen_normal(seed, i0, i0 + n, _vp(table), _vp(out),
                                                 _native.dtype_code(dtype), _stream_ptr(None)),
                  "dacsr_gen_normal")
    return out
