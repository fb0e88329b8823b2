"""ctypes binding of the C ABI in include/ridgepath_b200.h.

The library is the in-tree ``libridgepath_b200.so`` built by
``paper_1404_0466_b200.build``. There is no CPU fallback: if the library or a
CUDA device is missing, every compute entry point raises ``DeviceError``.
Status codes map onto the reference's exception taxonomy (errors.py):
negative -> UsageError (DimensionMismatch for shape errors), positive ->
DeviceError carrying the CUDA error string.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import DeviceError, DimensionMismatch

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libridgepath_b200.so")
HEADER_PATH = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "include", "ridgepath_b200.h"))

RP_METRIC_RMSE = 0
RP_METRIC_MISCLASS = 1

_vp = ctypes.c_void_p
_i = ctypes.c_int
_i64 = ctypes.c_int64
_d = ctypes.c_double
_sz = ctypes.c_size_t

# name -> (restype, argtypes); must list every function declared in include/ridgepath_b200.h
SIGNATURES = {
    "rp_version": (_i, []),
    "rp_last_error": (ctypes.c_char_p, []),
    "rp_launch_count": (ctypes.c_longlong, []),
    "rp_ozaki_fallbacks": (ctypes.c_longlong, []),
    "rp_tile_count": (_i64, [_i]),
    "rp_theta_size": (_i64, [_i, _i]),
    "rp_gram_workspace_size": (_sz, [_i, _i64, _i]),
    "rp_set_option": (_i, [ctypes.c_char_p, _i]),
    "rp_profile_ms": (ctypes.c_double, [ctypes.c_char_p]),
    "rp_gram_blocks": (_i, [_vp, _i64, _i64, _i, _i, _vp, _i64, _i, _vp, _vp, _vp, _vp]),
    "rp_col_sumsq": (_i, [_vp, _i64, _i64, _i, _i, _vp, _vp]),
    "rp_symmetrize": (_i, [_vp, _i, _i64, _i, _vp]),
    "rp_fold_systems": (_i, [_vp, _vp, _i, _i, _i, _vp, _i, _vp, _i, _vp, _vp, _vp]),
    "rp_potrf_workspace_size": (_sz, [_i, _i]),
    "rp_potrf_batched": (_i, [_vp, _i, _i64, _i, _vp, _vp, _vp]),
    "rp_fit_tiles": (_i, [_vp, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp]),
    "rp_fit_workspace_size": (_sz, [_i, _i, _i, _i]),
    "rp_eval_solve_workspace_size": (_sz, [_i, _i, _i, _i, _i]),
    "rp_eval_solve_plan": (_i, [_i, _i, _i, _i, _i, _vp]),
    "rp_eval_solve": (_i, [_vp, _i, _i, _i, _vp, _i, _vp, _i, _vp, _i64, _vp, _vp, _vp]),
    "rp_eval_materialize": (_i, [_vp, _i, _i, _d, _vp, _vp]),
    "rp_theta_export": (_i, [_vp, _i, _i, _vp, _i64, _vp, _vp]),
    "rp_theta_import": (_i, [_vp, _i, _i, _vp, _i64, _vp, _vp]),
    "rp_holdout_workspace_size": (_sz, [_i64, _i, _i, _i, _i]),
    "rp_holdout_direct": (_i, [_vp, _i64, _i64, _i64, _i, _vp, _i64, _i, _vp, _i64, _i64, _i, _i, _i, _vp, _vp,
                               _vp]),
    "rp_holdout_gram": (_i, [_vp, _i64, _vp, _i64, _vp, _i64, _i, _i, _vp, _i64, _i64, _i, _i, _vp, _i64, _i64, _vp,
                             _i64, _vp, _vp, _vp]),
    "rp_select": (_i, [_vp, _i, _i, _i, _vp, _vp, _vp]),
}

_lock = threading.Lock()
_lib = None


def load():
    """Load (once) and return the CDLL with typed signatures."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1404_0466_b200.build` "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error():
    msg = load().rp_last_error()
    return msg.decode() if msg else ""


def call(name, *args):
    """Invoke an rp_* entry point and map its status code onto exceptions."""
    rc = getattr(load(), name)(*args)
    if rc < 0:
        raise DimensionMismatch(f"{name}: {last_error()}")
    if rc > 0:
        raise DeviceError(f"{name}: CUDA error {rc}: {last_error()}")
    return rc


def query(name, *args):
    return getattr(load(), name)(*args)


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("a CUDA device is required: this package has no CPU fallback")
    load()


def ptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def host_ptr(a):
    """Pointer of a C-contiguous numpy array (host-side small parameter arrays)."""
    return ctypes.c_void_p(a.ctypes.data)


def stream():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
