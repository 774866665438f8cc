"""ctypes binding of the sm_100a C ABI (include/dacsr_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` into
``paper_2307_06305_b200/lib/libdacsr_b200.so``.  There is no fallback: if
it is missing or fails to load, every device entry point raises
``NativeLibraryMissing``.  ctypes.CDLL releases the GIL around each call,
matching the reference's ``nogil`` kernels (spmv/__init__.py:166-176).
"""

import ctypes
import os
import threading

from .errors import DeviceError, NativeLibraryMissing

# DACSR_LIB=checked selects the bounds-checked build (tests only)
_LIB_NAME = ("libdacsr_b200_checked.so" if os.environ.get("DACSR_LIB") == "checked"
             else "libdacsr_b200.so")
LIB_PATH = os.environ.get("DACSR_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "lib", _LIB_NAME)  # DACSR_LIB_PATH: A/B builds

# dtype / kind / order / variant codes (dacsr_b200.h)
I8, I16, I32, I64, F32, F64 = range(6)
F16, BF16 = 6, 7  # 16-bit values (extension; see include/dacsr_b200.h)
KIND_CSR, KIND_DA = 0, 1
ORDER_NAIVE, ORDER_MACC3, ORDER_STRIP4, ORDER_TREE = range(4)
VARIANT_CODES = {
    "auto": 0, "rowblock": 1, "scalar": 2, "vector2": 3, "vector4": 4, "vector8": 5,
    "vector16": 6, "warp": 7, "staged": 8, "wstream": 9, "sliced": 10, "sliced_pipe": 14, "tiled": 15,
}
STATUS = {0: "ok", 1: "invalid argument", 2: "unsupported dtype", 3: "unknown variant/order",
          4: "CUDA error", 5: "plan mismatch"}
ANALYZE_SCRATCH = 64
PLAN_NO_L2_PREFETCH = 1  # dacsr_plan_t.flags

_NP_CODE = {"int8": I8, "int16": I16, "int32": I32, "int64": I64, "float32": F32,
            "float64": F64, "float16": F16, "bfloat16": BF16}


def dtype_code(dtype):
    """Library dtype code of a numpy/torch dtype."""
    name = str(dtype).replace("torch.", "")
    try:
        return _NP_CODE[name]
    except KeyError:
        raise ValueError(f"dtype {dtype} has no library code") from None


class Matrix(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("rowptr_dtype", ctypes.c_int32),
                ("colids_dtype", ctypes.c_int32), ("values_dtype", ctypes.c_int32),
                ("nrows", ctypes.c_int64), ("ncols", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("rowptr", ctypes.c_void_p), ("colids", ctypes.c_void_p),
                ("values", ctypes.c_void_p)]


class Stats(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("entry_start", ctypes.c_int64), ("entry_end", ctypes.c_int64),
                ("max_len", ctypes.c_int64), ("empty_rows", ctypes.c_int64),
                ("mean_len", ctypes.c_double), ("cv_len", ctypes.c_double),
                ("scatter", ctypes.c_double)]


class Plan(ctypes.Structure):
    _fields_ = [("row_start", ctypes.c_int64), ("row_end", ctypes.c_int64),
                ("entry_base", ctypes.c_int64), ("entry_end", ctypes.c_int64),
                ("nblocks", ctypes.c_int64), ("cap", ctypes.c_int32),
                ("long_len", ctypes.c_int32), ("block_rows", ctypes.c_void_p),
                ("chunk_vcap", ctypes.c_int32), ("chunk_rows", ctypes.c_int32),
                ("n_complex", ctypes.c_int64), ("complex_chunks", ctypes.c_void_p),
                ("ctas_per_sm", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("slices", ctypes.c_void_p), ("tiles", ctypes.c_void_p)]


class Slices(ctypes.Structure):
    """dacsr_slices_t: the sliced device layout (32-row slices)."""
    _fields_ = [("row_start", ctypes.c_int64), ("row_end", ctypes.c_int64),
                ("nslices", ctypes.c_int64), ("total", ctypes.c_int64),
                ("max_len", ctypes.c_int32), ("medium_len", ctypes.c_int32),
                ("slice_ptr", ctypes.c_void_p), ("row_len", ctypes.c_void_p),
                ("inner", ctypes.c_void_p), ("values", ctypes.c_void_p),
                ("n_medium", ctypes.c_int64), ("m_nslices", ctypes.c_int64),
                ("m_total", ctypes.c_int64), ("medium_rows", ctypes.c_void_p),
                ("m_slice_ptr", ctypes.c_void_p), ("m_inner", ctypes.c_void_p),
                ("m_values", ctypes.c_void_p), ("n_long", ctypes.c_int64),
                ("long_rows", ctypes.c_void_p)]


class Tiles(ctypes.Structure):
    """dacsr_tiles_t: the band-tiled device layout (512-row groups x column tiles)."""
    _fields_ = [("row_start", ctypes.c_int64), ("row_end", ctypes.c_int64),
                ("ngroups", ctypes.c_int64), ("col0", ctypes.c_int64), ("cmax", ctypes.c_int64),
                ("tile_cols", ctypes.c_int32), ("step_group", ctypes.c_int32),
                ("total", ctypes.c_int64), ("nblocks", ctypes.c_int64),
                ("ent_ptr", ctypes.c_void_p), ("cnt_ptr", ctypes.c_void_p),
                ("tile_lo", ctypes.c_void_p), ("counts", ctypes.c_void_p),
                ("skip", ctypes.c_void_p), ("inner", ctypes.c_void_p),
                ("values", ctypes.c_void_p), ("n_ovf", ctypes.c_int64),
                ("ovf_rows", ctypes.c_void_p), ("masks", ctypes.c_void_p),
                ("order", ctypes.c_void_p)]


def typed_kernel_names():
    """The reference-named entry points declared by DACSR_DECLARE_KIND."""
    return [f"dacsr_{k}_{n}_{v}" for k in ("csr", "da")
            for v in ("f64", "f32")
            for n in ("naive", "shifted_base", "multi_acc3", "strip_mined4")]


_vp, _i32, _i64, _d, _u64 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double,
                             ctypes.c_uint64)
_P = ctypes.POINTER
_SIGNATURES = {
    "dacsr_version": ([], ctypes.c_char_p),
    "dacsr_last_error": ([], ctypes.c_char_p),
    "dacsr_analyze": ([_P(Matrix), _i64, _i64, _vp, _P(Stats), _vp], ctypes.c_int),
    "dacsr_plan_default_cap": ([_P(Stats), _i32, _i32], _i32),
    "dacsr_plan_nblocks": ([_P(Matrix), _i64, _i64, _i32], _i64),
    "dacsr_plan_build": ([_P(Matrix), _i64, _i64, _i64, _i64, _i32, _i32, _vp, _P(Plan), _vp],
                         ctypes.c_int),
    "dacsr_select_variant": ([_P(Stats), _i32], _i32),
    "dacsr_slices_count": ([_P(Matrix), _i64, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp],
                           ctypes.c_int),
    "dacsr_slices_fill": ([_P(Matrix), _P(Slices), _vp, _vp, _vp], ctypes.c_int),
    "dacsr_slices_medium_count": ([_P(Slices), _vp, _vp], ctypes.c_int),
    "dacsr_slices_medium_fill": ([_P(Matrix), _P(Slices), _vp], ctypes.c_int),
    "dacsr_tiles_extent": ([_P(Matrix), _i64, _i64, _vp, _vp], ctypes.c_int),
    "dacsr_tiles_count": ([_P(Matrix), _P(Tiles), _vp, _vp, _vp, _vp], ctypes.c_int),
    "dacsr_tiles_fill": ([_P(Matrix), _P(Tiles), _vp, _vp], ctypes.c_int),
    "dacsr_tiles_step_group": ([], _i32),
    "dacsr_tiles_max_cols": ([_i32], _i32),
    "dacsr_plan_chunks": ([_P(Matrix), _i64, _i64, _i32, _i32, _vp, _vp, _P(Plan), _vp],
                          ctypes.c_int),
    "dacsr_spmv": ([_P(Matrix), _P(Plan), _i32, _i32, _vp, _i64, _vp, _d, _d, _i64, _i64, _vp],
                   ctypes.c_int),
    "dacsr_spmv_dev_alpha": ([_P(Matrix), _P(Plan), _i32, _i32, _vp, _i64, _vp, _vp, _d, _i64,
                              _i64, _vp], ctypes.c_int),
    "dacsr_spmv_dev_alpha_sumsq": ([_P(Matrix), _P(Plan), _i32, _i32, _vp, _i64, _vp, _vp, _d,
                                    _i64, _i64, _vp, _vp], ctypes.c_int),
    "dacsr_scale": ([_vp, _i32, _i64, _d, _vp], ctypes.c_int),
    "dacsr_norm_alpha": ([_vp, _i64, _vp, _vp, _vp], ctypes.c_int),
    "dacsr_scale_dev": ([_vp, _i32, _i64, _vp, _vp], ctypes.c_int),
    "dacsr_spmv_host_streamed": ([_P(Matrix), _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _d, _d,
                                  _i64, _vp, _vp, _vp, _i32], ctypes.c_int),
    "dacsr_sumsq_chunks": ([_vp, _i32, _i64, _i64, _vp, _vp], ctypes.c_int),
    "dacsr_sumsq_from_groups": ([_vp, _i64, _i64, _vp, _vp], ctypes.c_int),
    "dacsr_sum_ordered": ([_vp, _i64, _vp, _vp], ctypes.c_int),
    "dacsr_bandwidth": ([_P(Matrix), _vp, _vp], ctypes.c_int),
    "dacsr_csr_to_da": ([_P(Matrix), _vp, _i32, _vp], ctypes.c_int),
    "dacsr_gen_banded_counts": ([_i64, _i64, _i32, _u64, _vp, _i64, _i64, _vp, _vp], ctypes.c_int),
    "dacsr_gen_banded_fill": ([_i64, _i64, _i32, _u64, _vp, _vp, _i64, _i64, _vp, _i32, _vp, _vp,
                               _vp, _i32, _vp], ctypes.c_int),
    "dacsr_gen_normal": ([_u64, _i64, _i64, _vp, _vp, _i32, _vp], ctypes.c_int),
    "dacsr_counts_to_rowptr": ([_vp, _i64, _vp, _i32, _vp, _P(ctypes.c_size_t), _vp],
                               ctypes.c_int),
    "dacsr_stream_probe": ([_vp, _i64, _i32, _i32, _vp, _vp], ctypes.c_int),
    "dacsr_host_adjacency": ([_i64, _vp, _vp, _vp, _vp], ctypes.c_int),
    "dacsr_host_rcm": ([_i64, _vp, _vp, _vp], ctypes.c_int),
    "dacsr_host_permute": ([_i64, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp], ctypes.c_int),
}
for _name in typed_kernel_names():
    _SIGNATURES[_name] = ([_vp, _vp, _vp, _vp, _vp, _d, _d, _i64, _i64, _vp], ctypes.c_int)

_lock = threading.Lock()
_lib = None


def lib():
    """The loaded library (raises NativeLibraryMissing if unavailable)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} is not built; run `python __graft_entry__.py` (build())")
            try:
                L = ctypes.CDLL(LIB_PATH)
            except OSError as exc:
                raise NativeLibraryMissing(f"cannot load {LIB_PATH}: {exc}") from exc
            for name, (args, res) in _SIGNATURES.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = res
            _lib = L
    return _lib


def check(status, what):
    """Map a non-zero C-ABI status to DeviceError (with the CUDA message)."""
    if status:
        detail = STATUS.get(status, "unknown status")
        if status == 4:
            detail += ": " + lib().dacsr_last_error().decode(errors="replace")
        raise DeviceError(status, f"{what} failed ({detail})")
