"""ctypes binding of the C ABI declared in include/shmem_b200.h.

This module is the whole Python<->native boundary: plain pointers, sizes and
ints, no torch types in any signature.  The shared library is built in-tree
(``python -m paper_2504_19442_b200._build``) and loading it is mandatory --
there is no CPU fallback on the product path; a missing library raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (
    AllocationError,
    ArgumentError,
    ConfigurationError,
    ShmemError,
    SynchronizationFault,
    UsageError,
)

LIB_NAME = "libshmem_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

SH_OK = 0
SH_ERR_ARG = 1
SH_ERR_ALLOC = 2
SH_ERR_TIMEOUT = 3
SH_ERR_CUDA = 4
SH_ERR_STATE = 5
SH_ERR_CONFIG = 6

SH_DTYPE_BF16 = 0
SH_DTYPE_FP16 = 1
SH_DTYPE_FP32 = 2
SH_DTYPE_I32 = 3
SH_DTYPE_I64 = 4
SH_PHASE_ALL = 0
SH_PHASE_COMM = 1
SH_PHASE_COMPUTE = 2
SH_SIG_SET = 0
SH_SIG_ADD = 1
SH_MAX_WORLD = 16

_c_int_p = ctypes.POINTER(ctypes.c_int)
_c_size_p = ctypes.POINTER(ctypes.c_size_t)
_c_u64_p = ctypes.POINTER(ctypes.c_uint64)
_vp = ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/shmem_b200.h one-to-one
SIGNATURES = {
    "sh_version": (ctypes.c_int, []),
    "sh_last_error": (ctypes.c_char_p, []),
    "sh_world_create": (ctypes.c_int, [ctypes.c_int, _c_int_p, ctypes.c_size_t, ctypes.c_int,
                                       ctypes.c_double, ctypes.POINTER(_vp)]),
    "sh_world_create_member": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_size_t, ctypes.c_int, ctypes.c_double,
                                              ctypes.POINTER(_vp)]),
    "sh_ipc_handle_size": (ctypes.c_int, []),
    "sh_export_ipc_handle": (ctypes.c_int, [_vp, _vp]),
    "sh_import_ipc_handles": (ctypes.c_int, [_vp, _vp]),
    "sh_world_destroy": (ctypes.c_int, [_vp]),
    "sh_alloc": (ctypes.c_int, [_vp, ctypes.c_size_t, ctypes.c_size_t, _c_size_p]),
    "sh_alloc_signals": (ctypes.c_int, [_vp, ctypes.c_int, _c_int_p]),
    "sh_heap_ptr": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_size_t,
                                   ctypes.POINTER(_vp)]),
    "sh_signal_ptr": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.POINTER(_vp)]),
    "sh_read_signals": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_u64_p]),
    "sh_reset_signals": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp]),
    "sh_fill_signals": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_uint64, _vp]),
    "sh_poll_error": (ctypes.c_int, [_vp, ctypes.c_int, _c_int_p]),
    "sh_clear_error": (ctypes.c_int, [_vp, ctypes.c_int]),
    "sh_ag_gemm": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp, ctypes.c_size_t, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_int, _c_int_p, ctypes.c_uint64, _vp]),
    "sh_gemm_rs": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp, ctypes.c_size_t, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_int, _c_int_p, ctypes.c_uint64, _vp]),
    "sh_ag_gemm_ex": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp, ctypes.c_size_t,
                                     ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, _c_int_p, ctypes.c_uint64,
                                     ctypes.c_int, ctypes.c_int, _vp]),
    "sh_gemm_rs_ex": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp, ctypes.c_size_t,
                                     ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, _c_int_p, ctypes.c_uint64,
                                     ctypes.c_int, _vp]),
    "sh_ag_subchunks": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_int_p]),
    "sh_putmem": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_size_t, _vp,
                                 ctypes.c_size_t, _vp]),
    "sh_getmem": (ctypes.c_int, [_vp, ctypes.c_int, _vp, ctypes.c_int, ctypes.c_size_t,
                                 ctypes.c_size_t, _vp]),
    "sh_signal_op": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_uint64, _vp]),
    "sh_signal_wait": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_uint64, _vp]),
    "sh_reduce_slots": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_size_t, ctypes.c_int,
                                       ctypes.c_size_t, ctypes.c_int, _vp, _vp]),
    "sh_multimem_st": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_size_t, ctypes.c_size_t, _vp]),
    "sh_multimem_ld_reduce": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, _vp,
                                             _vp]),
    "sh_trace_enable": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "sh_trace_read": (ctypes.c_int, [_vp, ctypes.c_int, _c_u64_p, ctypes.c_size_t, _c_int_p]),
    "sh_gemm_workspace_bytes": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                               _c_size_p]),
    "sh_gemm": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.c_int, _vp, ctypes.c_size_t, _vp]),
    "sh_set_tile_config": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "sh_set_schedule_config": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "sh_set_dynamic_tiles": (ctypes.c_int, [ctypes.c_int]),
    "sh_query_tile_config": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_int_p,
                                            _c_int_p, _c_int_p]),
    "sh_set_rank_solo": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]),
    "sh_stream_write_word": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]),
    "sh_stream_wait_word": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]),
    "sh_pace_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64,
                                    ctypes.POINTER(ctypes.c_uint64), ctypes.c_int, ctypes.c_double]),
}

_lock = threading.Lock()
_lib = None
_lib_path = None


def load(path: str | None = None):
    """Load (once) and return the C-ABI library; raises if it is missing, or
    if ``path`` names another library than the one already loaded."""
    global _lib, _lib_path
    if _lib is not None and path is None:  # hot path of every call: no lock
        return _lib
    with _lock:
        if _lib is not None:
            if path is not None and os.path.realpath(path) != _lib_path:
                raise ShmemError(f"native library already loaded from {_lib_path}, not {path}")
            return _lib
        p = path or os.environ.get("SHB_LIB") or LIB_PATH
        if not os.path.exists(p):
            raise ShmemError(
                f"native library {p} not built; run `python -m paper_2504_19442_b200._build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(p)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib_path = os.path.realpath(p)
        _lib = lib
        return lib


_EXC = {
    SH_ERR_ARG: ArgumentError,
    SH_ERR_ALLOC: AllocationError,
    SH_ERR_TIMEOUT: SynchronizationFault,
    SH_ERR_STATE: UsageError,
    SH_ERR_CONFIG: ConfigurationError,
}


def check(rc: int):
    """Map a C-ABI status code onto the reference exception taxonomy."""
    if rc == SH_OK:
        return
    msg = load().sh_last_error()
    msg = msg.decode() if msg else f"status {rc}"
    raise _EXC.get(rc, ShmemError)(msg)


def int_array(values):
    arr = (ctypes.c_int * len(values))(*values)
    return arr
