"""ctypes binding of the C ABI in ``include/widemod_b200.h``.

This is the "thin ctypes/C-ABI shim" between the Python operator API and the
sm_100a kernels.  It never falls back to a CPU path: if the library is
missing or fails to load, every call raises :class:`LibraryUnavailable`.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

from ._build import LIB_PATH, build

WM_OK = 0
WM_EINVAL = 1
WM_ECUDA = 2
WM_EUNSUPPORTED = 3
WM_ELENGTH = 4
WM_NTT_FWD, WM_NTT_INV, WM_NTT_FWD_INV, WM_NTT_COPY = 0, 1, 2, 3
WM_OP_VADD, WM_OP_VSUB, WM_OP_VMUL, WM_OP_AXPY = 0, 1, 2, 3
WM_FIELD_KARATSUBA, WM_FIELD_MONTGOMERY, WM_FIELD_BARRETT = 1, 2, 4
WM_REDUCTION_BARRETT, WM_REDUCTION_MONTGOMERY, WM_REDUCTION_SPECIAL_FORM = 0, 1, 2
REDUCTION_NAMES = {WM_REDUCTION_BARRETT: "barrett", WM_REDUCTION_MONTGOMERY: "montgomery",
                   WM_REDUCTION_SPECIAL_FORM: "special_form"}


class LibraryUnavailable(RuntimeError):
    """libwidemod_b200.so is not built or cannot be loaded."""


class DeviceError(RuntimeError):
    """A CUDA runtime failure reported by the library."""


class Unsupported(ValueError):
    """Width or size not built into the device library."""


_lock = threading.Lock()
_lib = None

_u32p = ctypes.POINTER(ctypes.c_uint32)
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int

# (name, restype, argtypes) for every symbol the header declares.
SIGNATURES = [
    ("wm_abi_version", _int, []),
    ("wm_last_error", ctypes.c_char_p, []),
    ("wm_limbs_for_bits", _int, [_int]),
    ("wm_supported_limbs", _int, [_int, ctypes.POINTER(_int), _int]),
    ("wm_field_create", _int, [_int, _u32p, _int, ctypes.POINTER(_vp)]),
    ("wm_field_create_ex", _int, [_int, _u32p, _int, _int, ctypes.POINTER(_vp)]),
    ("wm_field_destroy", _int, [_vp]),
    ("wm_field_info", _int, [_vp, ctypes.POINTER(_int), ctypes.POINTER(_int), ctypes.POINTER(_int)]),
    ("wm_field_reduction", _int, [_vp]),
    ("wm_vadd", _int, [_vp, _vp, _vp, _vp, _i64, _vp]),
    ("wm_vsub", _int, [_vp, _vp, _vp, _vp, _i64, _vp]),
    ("wm_vmul", _int, [_vp, _vp, _vp, _vp, _i64, _vp]),
    ("wm_axpy", _int, [_vp, _u32p, _vp, _vp, _vp, _i64, _vp]),
    ("wm_ntt_plan_create", _int, [_vp, _i64, _u32p, _u32p, _u32p, ctypes.POINTER(_vp)]),
    ("wm_ntt_plan_destroy", _int, [_vp]),
    ("wm_ntt_plan_info", _int, [_vp, ctypes.POINTER(_int), ctypes.POINTER(_int), _int]),
    ("wm_ntt_workspace_bytes", _i64, [_vp, _i64]),
    ("wm_ntt_forward", _int, [_vp, _vp, _vp, _i64, _vp, _vp]),
    ("wm_ntt_inverse", _int, [_vp, _vp, _vp, _i64, _vp, _vp]),
    ("wm_ntt_convolve", _int, [_vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    ("wm_ntt_pass", _int, [_vp, _int, _int, _vp, _vp, _i64, _vp]),
    ("wm_ntt_twiddles", _int, [_vp, _int, _i64, _vp, _vp]),
    ("wm_ntt_host", _int, [_vp, _int, _int, _int, _vp, _vp, _i64, _i64, _vp]),
    ("wm_blas_host", _int, [_vp, _int, _u32p, _int, _int, _vp, _vp, _vp, _i64, _i64, _vp]),
    ("wm_transpose", _int, [_int, _vp, _vp, _i64, _i64, _i64, _vp]),
    ("wm_scale_transpose", _int, [_vp, _vp, _vp, _vp, _i64, _i64, _vp]),
    ("wm_widemul", _int, [_int, _int, _vp, _vp, _vp, _i64, _vp]),
    ("wm_scale_transpose_scatter", _int, [_vp, _vp, _vp, _vp, ctypes.c_int, ctypes.c_int, _i64, _i64, _vp]),
    ("wm_twiddle_table_2d", _int, [_vp, _i64, _u32p, _i64, _i64, _i64, _vp, _vp]),
    ("wm_twiddle_factors", _int, [_vp, _i64, _u32p, _int, _vp, _vp, _vp]),
    ("wm_scale_transpose_fx", _int, [_vp, _vp, _vp, _vp, _int, _i64, _i64, _vp, _vp, _int, _int, _int, _i64, _i64,
                                     _vp]),
    ("wm_probe_imad_wide", _int, [_int, _i64, _vp, _vp, ctypes.POINTER(_i64)]),
    ("wm_ntt_pass_work", _int, [_vp, _int, _int, _i64, ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_double)]),
    ("wm_blas_work", _int, [_vp, _int, ctypes.POINTER(ctypes.c_double)]),
    ("wm_ref_to_limbs", _int, [_int, _int, _int, _vp, _vp, _i64, _vp]),
    ("wm_limbs_to_ref", _int, [_int, _int, _int, _vp, _vp, _i64, _vp]),
]


def load(path: str | Path | None = None, build_if_missing: bool = True):
    """Load (building first if needed) and return the ctypes library."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        import os
        env = os.environ.get("WM_LIB_PATH")  # A/B experiments only (tools/ab_timing.py)
        p = Path(path) if path else (Path(env) if env else LIB_PATH)
        if not p.exists():
            if not build_if_missing:
                raise LibraryUnavailable(f"{p} not built")
            try:
                build()
            except Exception as exc:  # no nvcc on this host, compile error
                raise LibraryUnavailable(f"cannot build {p.name}: {exc}") from exc
        try:
            lib = ctypes.CDLL(str(p))
        except OSError as exc:
            raise LibraryUnavailable(f"cannot load {p}: {exc}") from exc
        for name, res, args in SIGNATURES:
            if env and path is None and not hasattr(lib, name):
                continue  # A/B variant built before a diagnostic export existed
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.wm_abi_version() != 1:
            raise LibraryUnavailable("ABI version mismatch")
        if path is None:
            _lib = lib
        return lib


def check(rc: int, what: str = "") -> None:
    """Raise the Python exception matching a library status code."""
    if rc == WM_OK:
        return
    lib = load()
    msg = lib.wm_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == WM_EUNSUPPORTED:
        raise Unsupported(text)
    if rc == WM_ECUDA:
        raise DeviceError(text)
    raise ValueError(text)


def u32_array(limbs) -> ctypes.Array:
    arr = (ctypes.c_uint32 * len(limbs))(*limbs)
    return arr
