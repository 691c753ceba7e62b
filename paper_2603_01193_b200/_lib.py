"""ctypes binding of the C ABI in include/wos_b200.h (libwos_b200.so).

The shared library is built in-tree by ``paper_2603_01193_b200.build`` (or
``__graft_entry__.build()``). There is no CPU fallback: if the library or a CUDA
device is missing, every entry point raises ``WosUnavailableError``.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_char_p, c_double, c_int32, c_int64, c_uint32, c_uint64, c_void_p

__all__ = [
    "WosError",
    "WosUnavailableError",
    "WosProblem",
    "WosWalkConfig",
    "lib",
    "lib_path",
    "check",
    "MODE_REPLAY_F64",
    "MODE_REPLAY_F32",
    "MODE_NATIVE_F32",
]

MODE_REPLAY_F64 = 0
MODE_REPLAY_F32 = 1
MODE_NATIVE_F32 = 2

WOS_OK = 0
WOS_ERR_INVALID = 1
WOS_ERR_UNSUPPORTED = 2
WOS_ERR_CUDA = 3
WOS_ERR_EXTERIOR = 4
WOS_ERR_NOMEM = 5
WOS_ERR_MAJORANT = 6
ABI_VERSION = 4

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.environ.get("WOS_B200_LIB") or os.path.join(_HERE, "libwos_b200.so")


class WosError(RuntimeError):
    """A C-ABI call returned a non-zero status."""

    def __init__(self, status: int, message: str):
        super().__init__(f"wos status {status}: {message}")
        self.status = status
        self.message = message


class WosUnavailableError(RuntimeError):
    """The CUDA extension is not built or cannot run here (no CPU fallback)."""


class WosProblem(ctypes.Structure):
    _fields_ = [
        ("dim", c_int32),
        ("dom_kind", c_int32),
        ("n_dom", c_int32),
        ("dom", POINTER(c_double)),
        ("src_kind", c_int32),
        ("n_src", c_int32),
        ("src", POINTER(c_double)),
        ("bnd_kind", c_int32),
        ("n_bnd", c_int32),
        ("bnd", POINTER(c_double)),
        ("instance_key", c_uint64),
    ]


class WosWalkConfig(ctypes.Structure):
    _fields_ = [
        ("eps", c_double),
        ("max_steps", c_int64),
        ("antithetic", c_int32),
        ("mode", c_int32),
        ("rng_seed", c_uint64),
        ("sigma_bar", c_double),
        ("philox_rounds", c_int32),
        ("reserved", c_int32),
    ]


_P = c_void_p
_SIGNATURES = {
    "wos_abi_version": (c_int32, []),
    "wos_last_error": (c_char_p, []),
    "wos_context_create": (c_int32, [c_int32, POINTER(c_void_p)]),
    "wos_context_destroy": (None, [_P]),
    "wos_problem_set_create": (c_int32, [_P, POINTER(WosProblem), c_int32, POINTER(c_void_p)]),
    "wos_problem_set_destroy": (None, [_P]),
    "wos_check_interior": (c_int32, [_P, _P, c_int64, _P, _P, POINTER(c_int64), _P]),
    "wos_check_interior_host": (c_int32, [_P, _P, c_int64, _P, _P, POINTER(c_int64)]),
    "wos_walk_rows": (
        c_int32,
        [_P, _P, POINTER(WosWalkConfig), c_int64, _P, _P, _P, _P, _P, _P, _P, _P],
    ),
    "wos_walk_rows_host": (
        c_int32,
        [_P, _P, POINTER(WosWalkConfig), c_int64, _P, _P, _P, _P, _P, _P, _P],
    ),
    "wos_estimate": (
        c_int32,
        [_P, _P, POINTER(WosWalkConfig), c_int64, _P, _P, _P, c_int64, c_uint64, _P, _P, _P, _P],
    ),
    "wos_estimate_host": (
        c_int32,
        [_P, _P, POINTER(WosWalkConfig), c_int64, _P, _P, _P, c_int64, c_uint64, _P, _P, _P],
    ),
    "wos_context_exterior": (c_int32, [_P, _P, POINTER(c_int64)]),
    "wos_context_majorant": (c_int32, [_P, _P, POINTER(c_double)]),
    "wos_context_status": (c_int32, [_P, _P, POINTER(c_int64), POINTER(c_uint32), POINTER(c_double)]),
    "wos_context_counters": (c_int32, [_P, _P, POINTER(c_uint64), POINTER(c_uint64)]),
    "wos_cache_fold": (
        c_int32,
        [_P, c_int64, _P, _P, _P, _P, c_int64, _P, _P, _P, _P, _P],
    ),
    "wos_cache_targets": (c_int32, [_P, c_int64, _P, c_int64, _P, _P]),
    "wos_estimate_fold": (
        c_int32,
        [_P, _P, POINTER(WosWalkConfig), c_int64, _P, _P, _P, c_int64, c_uint64, _P, _P, _P,
         _P, _P, _P, _P],
    ),
    "wos_philox4x64": (c_int32, [_P, c_int64, _P, c_uint64, c_uint64, _P, _P]),
    "wos_philox4x32": (c_int32, [_P, c_int64, _P, c_uint32, c_uint32, _P, _P]),
    "wos_philox4x32_rounds": (c_int32, [_P, c_int64, _P, c_uint32, c_uint32, c_int32, _P, _P]),
    "wos_set_tuning": (c_int32, [_P, c_int32, c_int32]),
    "wos_set_refill_deferred": (c_int32, [_P, c_int32]),
    "wos_fastmath_probe": (c_int32, [_P, c_int64, _P, _P, _P, _P, _P, _P]),
    "wos_probe_peaks": (
        c_int32,
        [_P, POINTER(c_double), POINTER(c_double), POINTER(c_double), POINTER(c_int32)],
    ),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lock = threading.Lock()
_lib = None


def load_library(path: str | None = None) -> ctypes.CDLL:
    """Load libwos_b200.so and declare every C-ABI signature (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or lib_path
        if not os.path.exists(p):
            raise WosUnavailableError(
                f"{p} is missing: build the CUDA extension first "
                "(python -m paper_2603_01193_b200.build); there is no CPU fallback"
            )
        handle = ctypes.CDLL(p)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.wos_abi_version() != ABI_VERSION:
            raise WosUnavailableError("libwos_b200.so ABI version mismatch")
        if path is None:
            _lib = handle
        return handle


def lib() -> ctypes.CDLL:
    return load_library()


def last_error() -> str:
    msg = lib().wos_last_error()
    return msg.decode() if msg else ""


def check(status: int) -> None:
    if status != WOS_OK:
        raise WosError(int(status), last_error())
