"""ctypes binding of the C ABI in include/tide_b200.h (libtide_b200.so).

The product path has no fallback: if the library is missing or no CUDA device
is present, every op raises `NativeUnavailable` instead of computing anything
on the CPU.
"""

from __future__ import annotations

import ctypes
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
LIBPATH = os.path.join(_PKG, "_lib", "libtide_b200.so")

F32, F16, BF16 = 0, 1, 2
MODE_PER_TOKEN, MODE_BATCH_UNANIMOUS = 0, 1
NO_EXIT = -1
WORKSPACE_BYTES = 16 << 20
MAX_DECODE_ROWS = 16
ROUTE_INPUTS_READY = 1

_c_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_f32 = ctypes.c_float

# name -> (restype, argtypes), exactly the declarations of include/tide_b200.h
SIGNATURES = {
    "tide_version": (ctypes.c_char_p, []),
    "tide_last_error": (ctypes.c_char_p, []),
    "tide_sm_count": (ctypes.c_int, [ctypes.c_int]),
    "tide_workspace_bytes": (ctypes.c_size_t, []),
    "tide_workspace_init": (ctypes.c_int, [_c_p, _c_p]),
    "tide_route_uses_tensor_cores": (ctypes.c_int, [_i32, _i32, _i32]),
    "tide_route": (ctypes.c_int, [_c_p, _i64, _i64, _c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p,
                                  _i32, _f32, _f32, _i64, _c_p, _c_p, _c_p, _c_p, _c_p, _i32,
                                  _c_p, _c_p, _c_p, _c_p]),
    "tide_route_ex": (ctypes.c_int, [_c_p, _i64, _i64, _c_p, _i64, _i32, _i32, _c_p, _c_p,
                                     _c_p, _i32, _f32, _f32, _i64, _c_p, _c_p, _c_p, _c_p, _c_p,
                                     _i32, _c_p, _c_p, _c_p, ctypes.c_uint32, _c_p]),
    "tide_compact": (ctypes.c_int, [_c_p, _i64, _c_p, _c_p, _i32, _c_p, _i64, _i32, _i32, _c_p,
                                    _c_p, _c_p, _c_p, _c_p, _c_p, _c_p]),
    "tide_lm_head": (ctypes.c_int, [_c_p, _c_p, _i64, _i64, _i32, _c_p, _c_p, _i64, _i64, _c_p,
                                    _i64, _c_p]),
    "tide_select_project_split": (ctypes.c_int, [ctypes.POINTER(_c_p), _i32, _i64, _i32, _c_p,
                                                 _i64, _i32, _c_p, _f32, _c_p, _c_p, _i64, _c_p]),
    "tide_exit_encode": (ctypes.c_int, [_c_p, _i64, _c_p, _c_p]),
    "tide_exit_decode": (ctypes.c_int, [_c_p, _i64, _c_p, _c_p]),
    "tide_exit_project": (ctypes.c_int, [_c_p, _i64, _i32, _c_p, _i64, _c_p, _i32, _c_p, _f32,
                                         _i32, _c_p, _c_p, _i64, _c_p]),
    "tide_select_project": (ctypes.c_int, [ctypes.POINTER(_c_p), _i32, _i64, _i32, _c_p, _i64,
                                           _i32, _c_p, _f32, _c_p, _i64, _c_p]),
    "tide_cos_label": (ctypes.c_int, [ctypes.POINTER(_c_p), _i32, _c_p, _i64, _i32, _i64, _i32,
                                      _f32, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p]),
    "tide_route_tail": (ctypes.c_int, [ctypes.POINTER(_c_p), _i32, _i64, _i64, _i32, _i32, _c_p,
                                       _c_p, _i64, _i64, ctypes.POINTER(_c_p),
                                       ctypes.POINTER(_c_p), _i32, ctypes.POINTER(_i64), _f32,
                                       _f32, _c_p, _c_p, _c_p, ctypes.c_uint64, _c_p, _c_p]),
    "tide_route_tail_ex": (ctypes.c_int, [ctypes.POINTER(_c_p), _i32, _i64, _i64, _i32, _i32,
                                          _c_p, _c_p, _i64, _i64, _i64, ctypes.POINTER(_c_p),
                                          ctypes.POINTER(_c_p), _i32, ctypes.POINTER(_i64), _f32,
                                          _f32, _c_p, _c_p, _c_p, ctypes.c_uint64, _c_p, _c_p]),
    "tide_route_multi": (ctypes.c_int, [ctypes.POINTER(_c_p), _i32, _i64, _i64, _c_p, _i64, _i32,
                                        _i32, _c_p, ctypes.POINTER(_c_p), ctypes.POINTER(_c_p),
                                        _i32, ctypes.POINTER(_i64), _f32, _f32, _c_p, _c_p, _c_p,
                                        _c_p]),
    "tide_capture_cond_create": (ctypes.c_int, [_c_p, ctypes.POINTER(ctypes.c_uint64)]),
    "tide_capture_cond_open": (ctypes.c_int, [_c_p, ctypes.c_uint64, ctypes.POINTER(_c_p)]),
    "tide_capture_cond_close": (ctypes.c_int, [_c_p]),
    "tide_train_act": (ctypes.c_int, [_c_p, _i64, _i32, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p,
                                      _c_p, _c_p]),
    "tide_adam_step": (ctypes.c_int, [_c_p, _c_p, _c_p, _c_p, _i64, _f32, _f32, _f32, _f32,
                                      _c_p, _c_p, _i64, _f32, _f32, _f32, _f32, _c_p]),
    "tide_route_decode": (ctypes.c_int, [ctypes.POINTER(_c_p), _i32, _i64, _i64, _i32, _i32,
                                         ctypes.POINTER(_c_p), ctypes.POINTER(_c_p), _i32,
                                         ctypes.POINTER(_i64), _f32, _f32, _i64, _i32, _c_p,
                                         _c_p, _c_p, _c_p, _c_p, _c_p]),
    "tide_route_decode_ex": (ctypes.c_int, [ctypes.POINTER(_c_p), _i32, _i64, _i64, _i32, _i32,
                                            ctypes.POINTER(_c_p), ctypes.POINTER(_c_p), _i32,
                                            ctypes.POINTER(_i64), _f32, _f32, _i64, _i32, _c_p,
                                            _c_p, _c_p, _c_p, _c_p, _c_p, _c_p]),
    "tide_decode_packed_bytes": (ctypes.c_size_t, [_i32, _i32, _i32]),
    "tide_decode_pack_weights": (ctypes.c_int, [ctypes.POINTER(_c_p), _i32, _i32, _i32, _i32,
                                                _c_p, _c_p]),
}


class NativeUnavailable(RuntimeError):
    """The CUDA library (or a CUDA device) is missing; there is no CPU fallback."""


class NativeError(RuntimeError):
    """A kernel launch or argument check failed inside libtide_b200."""


_lib = None
_lock = threading.Lock()


def _check_fresh() -> None:
    """The library must match the sources next to it (a stale .so would run
    old kernels against new host code)."""
    from . import build as _build
    stamp = os.path.join(os.path.dirname(LIBPATH), "build.stamp")
    if not os.path.exists(stamp):
        return
    with open(stamp) as fh:
        if fh.read().strip() != _build._fingerprint():
            raise NativeUnavailable(
                f"{LIBPATH} is stale (sources changed since it was built); run "
                "`python -m paper_2603_21365_b200.build`")


def load(path: str = LIBPATH):
    """Load (once) and return the ctypes library with typed signatures."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise NativeUnavailable(
                    f"{path} not built; run `python -m paper_2603_21365_b200.build` "
                    "(there is no CPU fallback)")
            if path == LIBPATH and os.environ.get("TIDE_ALLOW_STALE") != "1":
                _check_fresh()
            lib = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().tide_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed ({rc}): {msg}")


def ptr_array(ptrs):
    arr = (_c_p * len(ptrs))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def i64_array(vals):
    arr = (_i64 * len(vals))()
    for i, v in enumerate(vals):
        arr[i] = int(v)
    return arr
