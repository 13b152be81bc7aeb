"""The C-ABI library builds for sm_100a, loads, and exports every symbol the
public header declares.  Only host-only entry points are called here (no
kernel launches, no CUDA context needed)."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

from paper_2501_07535_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "widemod_b200.h"


def declared_symbols() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(wm_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    return _lib.load()


def test_header_symbols_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(lib, name), name
    assert sorted(n for n, _, _ in _lib.SIGNATURES) == syms


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    assert out.returncode == 0 and "sm_100a" in out.stdout


def test_host_only_entry_points(lib):
    assert lib.wm_abi_version() == 1
    assert lib.wm_limbs_for_bits(256) == 8
    assert lib.wm_limbs_for_bits(384) == 12
    assert lib.wm_limbs_for_bits(768) == 24
    assert lib.wm_limbs_for_bits(16) == 1
    buf = (ctypes.c_int * 32)()
    m = lib.wm_supported_limbs(1, buf, 32)
    assert {1, 2, 4, 8, 12, 16, 24, 32} <= set(buf[:m])


def test_field_create_validation(lib):
    h = ctypes.c_void_p()
    q = (ctypes.c_uint32 * 8)(*([0xFFFFFF7F] + [0xFFFFFFFF] * 6 + [0x0FFFFFFF]))  # 2^252 - 129
    assert lib.wm_field_create(256, q, 8, ctypes.byref(h)) == _lib.WM_OK
    b, k, s = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    assert lib.wm_field_info(h, ctypes.byref(b), ctypes.byref(k), ctypes.byref(s)) == 0
    assert (b.value, k.value, s.value) == (256, 8, 0)
    lib.wm_field_destroy(h)
    # q = 500 at width 13 (reference test_kernels.py:31-33): normalisation shift 19
    q500 = (ctypes.c_uint32 * 1)(500)
    assert lib.wm_field_create(13, q500, 1, ctypes.byref(h)) == 0
    assert lib.wm_field_info(h, ctypes.byref(b), ctypes.byref(k), ctypes.byref(s)) == 0
    assert (k.value, s.value) == (1, 19)
    lib.wm_field_destroy(h)
    one = (ctypes.c_uint32 * 1)(1)
    assert lib.wm_field_create(16, one, 1, ctypes.byref(h)) == _lib.WM_EINVAL
    assert b"exceed" in lib.wm_last_error()
    big = (ctypes.c_uint32 * 1)(0xFFFFFFFF)
    assert lib.wm_field_create(32, big, 1, ctypes.byref(h)) == _lib.WM_EINVAL
    assert lib.wm_field_create(4000, one, 1, ctypes.byref(h)) == _lib.WM_EUNSUPPORTED


def _limbs(v: int, k: int):
    return (ctypes.c_uint32 * k)(*[(v >> (32 * i)) & 0xFFFFFFFF for i in range(k)])


def test_full_width_and_padded_field_creation(lib):
    """Host-side field setup (no device work): full-width (Montgomery)
    fields, their validation, and widths padded to a built limb count."""
    h = ctypes.c_void_p()
    b, k, s = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    secp = 2**256 - 2**32 - 977
    assert lib.wm_field_create_ex(256, _limbs(secp, 8), 8, _lib.WM_FIELD_MONTGOMERY, ctypes.byref(h)) == 0
    assert lib.wm_field_info(h, ctypes.byref(b), ctypes.byref(k), ctypes.byref(s)) == 0
    assert (b.value, k.value, s.value) == (256, 8, 0)  # top bit set: full-width Barrett shift 0
    lib.wm_field_destroy(h)
    # the Barrett path keeps the reference range
    assert lib.wm_field_create_ex(256, _limbs(secp, 8), 8, 0, ctypes.byref(h)) == _lib.WM_EINVAL
    # Montgomery needs an odd modulus; Karatsuba applies to Barrett fields only
    assert lib.wm_field_create_ex(256, _limbs(secp + 1, 8), 8, _lib.WM_FIELD_MONTGOMERY, ctypes.byref(h)) == _lib.WM_EINVAL
    assert lib.wm_field_create_ex(256, _limbs(secp, 8), 8, 3, ctypes.byref(h)) == _lib.WM_EINVAL
    # 640 bits (20 limbs, no kernels of its own) runs zero-padded to 24 limbs
    assert lib.wm_limbs_for_bits(640) == 24 and lib.wm_limbs_for_bits(512) == 16
    q640 = 2**636 - 3 * 2**400 - 1  # odd, reference range
    assert lib.wm_field_create_ex(640, _limbs(q640, 20), 20, 0, ctypes.byref(h)) == 0
    assert lib.wm_field_info(h, ctypes.byref(b), ctypes.byref(k), ctypes.byref(s)) == 0
    assert k.value == 24
    lib.wm_field_destroy(h)
    assert lib.wm_field_create_ex(640, _limbs(q640 + 1, 20), 20, 0, ctypes.byref(h)) == _lib.WM_EUNSUPPORTED


def test_blas_work_model(lib):
    """wm_blas_work (host only): word products per element in each field
    arithmetic, against hand counts of the templates in wm_limb.cuh."""
    def work(bits, q, flags, op):
        k = lib.wm_limbs_for_bits(bits)
        h = ctypes.c_void_p()
        assert lib.wm_field_create_ex(bits, _limbs(q, k), k, flags, ctypes.byref(h)) == _lib.WM_OK
        wp = ctypes.c_double()
        rc = lib.wm_blas_work(h, op, ctypes.byref(wp))
        lib.wm_field_destroy(h)
        return rc, wp.value

    KA, BA, MO = 1, 4, 2  # WM_FIELD_KARATSUBA / BARRETT / MONTGOMERY
    q256, q768 = (1 << 252) - 129, (1 << 764) - 393
    assert work(256, q256, 0, _lib.WM_OP_VADD) == (0, 0.0)
    assert work(256, q256, 0, _lib.WM_OP_VMUL) == (0, 64 + 8 + 2)          # schoolbook + two folds
    assert work(256, q256, KA, _lib.WM_OP_AXPY) == (0, 48 + 8 + 2)         # one Karatsuba level
    assert work(256, q256, KA | BA, _lib.WM_OP_VMUL) == (0, 48 + 43 + 28 + 4)  # Barrett: full + hi + lo
    assert work(768, q768, KA, _lib.WM_OP_VMUL) == (0, 324 + 24 + 2)       # two Karatsuba levels
    assert work(768, q768, KA | BA, _lib.WM_OP_VMUL) == (0, 324 + 323 + 276 + 12)
    assert work(256, (1 << 255) - 19, MO, _lib.WM_OP_VMUL)[0] == _lib.WM_EUNSUPPORTED
