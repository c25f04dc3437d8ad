"""ctypes binding of libsldb200.so (include/sldb200.h).

The product path is Python -> ctypes -> CUDA.  There is no CPU fallback:
if the shared library is missing or no CUDA device is visible, every call
that needs the device raises `NativeUnavailable` (a RuntimeError).
"""
import ctypes
import os
import threading

import numpy as np

from . import _build

LIB_PATH = os.environ.get("SLD_LIB", _build.LIB)  # SLD_LIB: experiment builds only

SLD_OK = 0
SLD_E_ARG = -1
SLD_E_CUDA = -2
SLD_E_BOUND = -3
SLD_E_TIMEOUT = -4
SLD_E_FORMAT = -5
SLD_E_MAGIC = -6
SLD_E_TRUNC = -7
SLD_E_PROTOCOL = -8
SLD_GRID_BLOB = 128

# every symbol include/sldb200.h declares (checked by tests/test_native_abi.py)
EXPORTS = [
    "sld_version", "sld_last_error", "sld_device_count", "sld_die_map",
    "sld_ctx_create", "sld_ctx_destroy", "sld_ctx_sync", "sld_ctx_set_stream", "sld_add_mod",
    "sld_vec_read_rows", "sld_lincomb", "sld_vec_nonzero",
    "sld_mat_create", "sld_mat_create_chains", "sld_mat_destroy", "sld_mat_info",
    "sld_vec_create", "sld_vec_create_chains", "sld_vec_destroy", "sld_vec_upload_planes", "sld_vec_download_planes",
    "sld_vec_upload_limbs", "sld_vec_download_limbs", "sld_vec_device_ptr",
    "sld_vec_upload_planes_chains", "sld_vec_download_planes_chains",
    "sld_lcset_create", "sld_lcset_apply", "sld_lcset_apply_batch", "sld_lcset_create_slots", "sld_lcset_destroy",
    "sld_spmv", "sld_spmv_async", "sld_spmv_planes", "sld_krylov_unit",
    "sld_xblock_create", "sld_xblock_destroy", "sld_krylov_dense",
    "sld_bench_spmv", "sld_bench_spmv_samples", "sld_corpus_rows", "sld_corpus_fill",
    "sld_sldm_info", "sld_sldm_read", "sld_sldm_write", "sld_sldv_write", "sld_sldv_info", "sld_sldv_read",
    "sld_split_block", "sld_mat_mksol_bind", "sld_spmv_mksol", "sld_spmv_add",
    "sld_grid_create", "sld_grid_blob", "sld_grid_connect", "sld_grid_set_timeout", "sld_grid_set_projection",
    "sld_grid_load", "sld_grid_read", "sld_grid_launch", "sld_grid_wait", "sld_grid_iterate", "sld_grid_terms",
    "sld_grid_set_epoch", "sld_grid_info", "sld_grid_destroy",
]


class NativeUnavailable(RuntimeError):
    """libsldb200.so could not be loaded or no CUDA device is usable."""


class BoundError(AssertionError):
    """Exactness bound exceeded (the reference raises AssertionError /
    ContractViolation for the same condition, vecops.py:407,414)."""


class GridProtocolError(RuntimeError):
    """A grid node published the wrong iteration: stale or restarted
    (the reference's gridmv.GridProtocolError, gridmv.py:46-47)."""


class GridTimeoutError(RuntimeError):
    """A grid barrier / expected message never completed: a node stopped
    (the reference's gridmv.GridTimeoutError, gridmv.py:50-51)."""


_lib = None
_lock = threading.Lock()


def load(build_if_missing=False):
    """Load the shared library (raises NativeUnavailable if absent)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            if build_if_missing:
                _build.build()
            else:
                raise NativeUnavailable(
                    f"{LIB_PATH} is missing; build it with `python -m paper_1402_3661_b200._build` "
                    "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32, u64p = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        pp = ctypes.POINTER(ctypes.c_void_p)
        sig = {
            "sld_version": ([], i32),
            "sld_last_error": ([], ctypes.c_char_p),
            "sld_device_count": ([vp], i32),
            "sld_die_map": ([i32, vp, vp, vp], i32),
            "sld_ctx_create": ([i32, vp, i32, pp], i32),
            "sld_ctx_destroy": ([vp], i32),
            "sld_ctx_sync": ([vp], i32),
            "sld_ctx_set_stream": ([vp, ctypes.c_uint64], i32),
            "sld_add_mod": ([vp, vp, i32, ctypes.c_uint64, i64], i32),
            "sld_vec_read_rows": ([vp, vp, i32, vp], i32),
            "sld_lincomb": ([vp, vp, vp, i32, ctypes.c_uint64, ctypes.c_uint64, i64], i32),
            "sld_vec_nonzero": ([vp, vp], i32),
            "sld_mat_create": ([vp, i64, i64, vp, vp, vp, vp, i64, vp, vp, i32, vp, i64, pp], i32),
            "sld_mat_create_chains": ([vp, i32, i64, i64, vp, vp, vp, vp, i64, vp, vp, i32, vp, i64, pp], i32),
            "sld_mat_destroy": ([vp], i32),
            "sld_mat_info": ([vp, vp], i32),
            "sld_vec_create": ([vp, i64, pp], i32),
            "sld_vec_create_chains": ([vp, i64, i32, pp], i32),
            "sld_vec_destroy": ([vp], i32),
            "sld_vec_upload_planes": ([vp, u64p, i64, i32], i32),
            "sld_vec_download_planes": ([vp, u64p, i64, i32], i32),
            "sld_vec_upload_limbs": ([vp, vp, i64], i32),
            "sld_vec_upload_planes_chains": ([vp, vp, i64, i32], i32),
            "sld_lcset_create": ([vp, vp, i32, i64, pp], i32),
            "sld_lcset_apply": ([vp, vp, ctypes.c_uint64, ctypes.c_uint64], i32),
            "sld_lcset_apply_batch": ([vp, vp, i32, vp], i32),
            "sld_lcset_create_slots": ([vp, vp, i32, vp], i32),
            "sld_lcset_destroy": ([vp], i32),
            "sld_vec_download_planes_chains": ([vp, vp, i64, i32], i32),
            "sld_vec_download_limbs": ([vp, vp, i64], i32),
            "sld_vec_device_ptr": ([vp, vp, vp], i32),
            "sld_spmv": ([vp, vp, vp], i32),
            "sld_spmv_async": ([vp, vp, vp], i32),
            "sld_spmv_planes": ([vp, vp, vp, i32], i32),
            "sld_krylov_unit": ([vp, vp, vp, i32, i64, vp], i32),
            "sld_xblock_create": ([vp, vp, i32, i64, pp], i32),
            "sld_xblock_destroy": ([vp], i32),
            "sld_krylov_dense": ([vp, vp, vp, i64, vp], i32),
            "sld_bench_spmv": ([vp, vp, i64, i32, vp, vp], i32),
            "sld_bench_spmv_samples": ([vp, vp, i64, i32, i64, vp, vp, vp], i32),
            "sld_sldm_info": ([ctypes.c_char_p, i32, vp, vp, i32], i32),
            "sld_sldm_read": ([ctypes.c_char_p, i32, vp, vp, vp, vp, vp, vp, vp, vp], i32),
            "sld_sldm_write": ([ctypes.c_char_p, i64, i64, vp, i32, vp, vp, vp, vp, i64, vp, vp, i32, vp, vp],
                               i32),
            "sld_sldv_write": ([ctypes.c_char_p, i32, vp, i32, i64, i64, vp, i32], i32),
            "sld_sldv_info": ([ctypes.c_char_p, i32, vp, vp, i32], i32),
            "sld_sldv_read": ([ctypes.c_char_p, vp, i32], i32),
            "sld_corpus_rows": ([i64, i64, ctypes.c_double, ctypes.c_uint64, vp], i32),
            "sld_corpus_fill": ([i64, i64, ctypes.c_double, ctypes.c_double, i64, ctypes.c_uint64,
                                 vp, vp, vp, vp, i32], i32),
            "sld_mat_mksol_bind": ([vp, vp, i32], i32),
            "sld_spmv_mksol": ([vp, vp, vp, vp], i32),
            "sld_spmv_add": ([vp, vp, vp, vp], i32),
            "sld_grid_create": ([vp, i32, i32, i32, i64, vp], i32),
            "sld_grid_blob": ([vp, vp], i32),
            "sld_grid_connect": ([vp, vp], i32),
            "sld_grid_set_timeout": ([vp, ctypes.c_double], i32),
            "sld_grid_set_projection": ([vp, vp, i32, i64, vp], i32),
            "sld_grid_load": ([vp, vp], i32),
            "sld_grid_read": ([vp, vp], i32),
            "sld_grid_launch": ([vp, i64], i32),
            "sld_grid_wait": ([vp], i32),
            "sld_grid_iterate": ([vp, i64], i32),
            "sld_grid_terms": ([vp, vp, vp], i32),
            "sld_grid_set_epoch": ([vp, i64], i32),
            "sld_grid_info": ([vp, vp], i32),
            "sld_grid_destroy": ([vp], i32),
            "sld_split_block": ([i64, vp, vp, i32, vp, vp, i64, vp, vp, i64, i32, i32, i32, i32, vp, vp, vp, i32],
                                i64),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return _lib


def check(rc):
    """Map a C-ABI status to the reference's exception types."""
    if rc == SLD_OK:
        return
    msg = load().sld_last_error().decode(errors="replace")
    if rc == SLD_E_ARG:
        raise ValueError(msg)
    if rc == SLD_E_BOUND:
        raise BoundError(msg)
    if rc == SLD_E_TIMEOUT:
        raise GridTimeoutError(msg)
    if rc == SLD_E_PROTOCOL:
        raise GridProtocolError(msg)
    raise RuntimeError(f"libsldb200: {msg}")


def device_count():
    n = ctypes.c_int(0)
    rc = load().sld_device_count(ctypes.byref(n))
    if rc != SLD_OK:
        return 0
    return n.value


def die_map(device=0):
    """(map[256] of %smid -> die, SMs on die 0, SMs on die 1), or None when
    the probe is ambiguous (the SpMV then runs without the die split)."""
    import numpy as np
    m = np.zeros(256, dtype=np.uint8)
    n0, n1 = ctypes.c_int(0), ctypes.c_int(0)
    rc = load().sld_die_map(int(device), m.ctypes.data, ctypes.byref(n0), ctypes.byref(n1))
    if rc != SLD_OK:
        return None
    return m, n0.value, n1.value


def ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else ctypes.c_void_p(0)


def c64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def c32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def cu32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)
