"""The C-ABI library loads on a CPU-only host and exports every symbol the
public header declares (no device compute is issued here)."""

import ctypes
import os
import re

from conftest import ROOT
from paper_2307_06305_b200 import _native

HEADER = os.path.join(ROOT, "include", "dacsr_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(dacsr_\w+)\s*\(", text, flags=re.M))
    names.discard("dacsr_")
    return sorted(n for n in names if not n.startswith("dacsr_##")) + _native.typed_kernel_names()


def test_header_functions_found():
    names = declared_functions()
    assert "dacsr_spmv" in names and "dacsr_host_rcm" in names
    assert "dacsr_da_naive_f64" in names and len(names) >= 36


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_bindings_cover_header():
    assert set(declared_functions()) <= set(_native._SIGNATURES)


def test_version_and_error_string():
    L = _native.lib()
    assert b"sm_100a" in L.dacsr_version()
    assert L.dacsr_last_error() is not None


def test_arg_validation_without_device():
    """Argument errors are reported before any CUDA call."""
    L = _native.lib()
    assert L.dacsr_spmv(None, None, 0, 0, None, 0, None, 1.0, 0.0, 0, 1, None) == 1
    m = _native.Matrix(1, 2, 1, 5, 4, 4, 5, None, None, None)
    assert L.dacsr_spmv(ctypes.byref(m), None, 0, 7, None, 0, ctypes.c_void_p(8), 1.0, 0.0, 0, 4,
                        None) == 1  # null rowptr
    assert L.dacsr_plan_nblocks(ctypes.byref(m), 3, 100, 32) == 4
    st = _native.Stats(4, 5, 0, 5, 2, 0, 1.25, 0.3)
    cap = L.dacsr_plan_default_cap(ctypes.byref(st), _native.F64, _native.I16)
    assert cap % 16 == 0 and cap >= 512


def test_slices_arg_validation_without_device():
    """The sliced-layout builder rejects bad arguments before any CUDA call."""
    L = _native.lib()
    m = _native.Matrix(_native.KIND_DA, _native.I32, _native.I16, _native.F64, 64, 64, 100,
                       None, None, None)
    # null rowptr / bad max_len / medium_len < max_len / bad row range
    assert L.dacsr_slices_count(ctypes.byref(m), 0, 64, 4, 8, None, None, None, None, None) == 1
    m.rowptr = 16
    assert L.dacsr_slices_count(ctypes.byref(m), 0, 64, 0, 8, None, None, None, None, None) == 1
    assert L.dacsr_slices_count(ctypes.byref(m), 0, 64, 9, 8, None, None, None, None, None) == 1
    assert L.dacsr_slices_count(ctypes.byref(m), 0, 65, 4, 8, None, None, None, None, None) == 1
    assert L.dacsr_slices_count(ctypes.byref(m), 0, 64, 4, 255, None, None, None, None, None) == 1
    sl = _native.Slices()
    assert L.dacsr_slices_fill(ctypes.byref(m), ctypes.byref(sl), None, None, None) == 1
    assert L.dacsr_slices_medium_fill(ctypes.byref(m), ctypes.byref(sl), None) == 1
    # a SLICED launch without a plan / without slices is a plan error
    p = _native.Plan()
    x = ctypes.c_void_p(8)
    m.colids, m.values = 32, 64
    assert L.dacsr_spmv(ctypes.byref(m), None, _native.VARIANT_CODES["sliced"], 0, x, 0, x,
                        1.0, 0.0, 0, 64, None) == 5
    assert L.dacsr_spmv(ctypes.byref(m), ctypes.byref(p), _native.VARIANT_CODES["sliced"], 0, x,
                        0, x, 1.0, 0.0, 0, 64, None) == 5


def test_generator_and_fused_norm_arg_validation_without_device():
    """A row draws up to kmax - 1 distinct non-zero offsets from [-b, b]: the
    generator refuses kmax - 1 > 2b (it would never finish) before any CUDA
    call; so do the fused-norm entry points on bad arguments."""
    L = _native.lib()
    p = ctypes.c_void_p(8)
    assert L.dacsr_gen_banded_counts(512, 1, 4, 1, p, 0, 512, p, None) == 1
    assert L.dacsr_gen_banded_counts(512, 1, 65, 1, p, 0, 512, p, None) == 1
    assert L.dacsr_gen_banded_fill(512, 1, 4, 1, p, p, 0, 512, p, _native.I32, p, None, p,
                                   _native.F64, None) == 1
    # chunk not a multiple of 512 / null pointers
    assert L.dacsr_sumsq_from_groups(p, 4096, 1000, p, None) == 1
    assert L.dacsr_sumsq_from_groups(None, 4096, 1024, p, None) == 1
    assert L.dacsr_sumsq_from_groups(None, 0, 1024, None, None) == 0
    m = _native.Matrix(_native.KIND_DA, _native.I32, _native.I16, _native.F64, 1024, 1024, 100,
                       16, 32, 64)
    # group sums exist on the TILED kernel only; null group buffer
    assert L.dacsr_spmv_dev_alpha_sumsq(ctypes.byref(m), None, _native.VARIANT_CODES["sliced"], 0,
                                        p, 0, p, p, 0.0, 0, 1024, p, None) == 3
    assert L.dacsr_spmv_dev_alpha_sumsq(ctypes.byref(m), None, _native.VARIANT_CODES["tiled"], 0,
                                        p, 0, p, p, 0.0, 0, 1024, None, None) == 1
