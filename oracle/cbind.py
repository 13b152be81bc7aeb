"""TEST INFRASTRUCTURE ONLY — ctypes binding of oracle/liboracle.so (the C
restatement in oracle/ntt_oracle.c).  Inputs/outputs are numpy uint32 arrays
[count, K] in the device layout (little-endian 32-bit limbs)."""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

from .bigint import compute_barrett

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"

_lib = None


def build() -> Path:
    src = HERE / "ntt_oracle.c"
    if LIB.exists() and LIB.stat().st_mtime >= src.stat().st_mtime:
        return LIB
    subprocess.run(["make", "-C", str(HERE), "liboracle.so"], check=True, capture_output=True)
    return LIB


def load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(str(LIB))
        vp, i64, i = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        lib.or_field_size.restype = i
        lib.or_field_init.argtypes = [vp, i, i, vp, vp, i, i]
        lib.or_vector.argtypes = [vp, i, vp, vp, vp, vp, i64]
        lib.or_powers.argtypes = [vp, vp, i64, vp]
        lib.or_ntt.argtypes = [vp, vp, i64, vp, vp, i64]
        lib.or_ntt_points.argtypes = [vp, vp, i64, vp, vp, i, vp]
        _lib = lib
    return _lib


def _limbs(v: int, K: int) -> np.ndarray:
    return np.frombuffer(int(v).to_bytes(4 * K, "little"), dtype="<u4").copy()


def _p(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"] and a.dtype == np.uint32
    return a.ctypes.data


class OracleField:
    """The reference's Barrett arithmetic mod q at interface width `width`."""

    def __init__(self, q: int, width: int):
        self.lib = load()
        self.q, self.width = q, width
        self.K = (width + 31) // 32
        _, mu, s1, s2 = compute_barrett(q, width)
        self._buf = ctypes.create_string_buffer(self.lib.or_field_size())
        qa, mua = _limbs(q, self.K), _limbs(mu, self.K)
        rc = self.lib.or_field_init(self._buf, self.K, width, _p(qa), _p(mua), s1, s2)
        assert rc == 0

    def vector(self, kind: str, x: np.ndarray, y: np.ndarray, scalar: int = 0) -> np.ndarray:
        code = {"vadd": 0, "vsub": 1, "vmul": 2, "axpy": 3}[kind]
        x = np.ascontiguousarray(x, dtype=np.uint32)
        y = np.ascontiguousarray(y, dtype=np.uint32)
        out = np.empty_like(x)
        a = _limbs(scalar, self.K)
        self.lib.or_vector(self._buf, code, _p(a), _p(x), _p(y), _p(out), x.shape[0])
        return out

    def powers(self, base: int, count: int) -> np.ndarray:
        out = np.empty((count, self.K), dtype=np.uint32)
        b = _limbs(base, self.K)
        self.lib.or_powers(self._buf, _p(b), count, _p(out))
        return out

    def ntt(self, x: np.ndarray, n: int, root: int, n_inv: int | None = None) -> np.ndarray:
        """run_ntt on x[batch*n, K]; n_inv given -> inverse (root = root_inv)."""
        v = np.ascontiguousarray(x, dtype=np.uint32).copy()
        batch = v.shape[0] // n
        tw = self.powers(root, max(1, n // 2))
        ni = _limbs(n_inv, self.K) if n_inv is not None else None
        self.lib.or_ntt(self._buf, _p(tw), n, _p(ni) if ni is not None else None, _p(v), batch)
        return v

    def ntt_points(self, x: np.ndarray, root: int, ks) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.uint32)
        kk = np.ascontiguousarray(np.asarray(ks, dtype=np.int64))
        out = np.empty((len(kk), self.K), dtype=np.uint32)
        r = _limbs(root, self.K)
        self.lib.or_ntt_points(self._buf, _p(x), x.shape[0], _p(r), kk.ctypes.data, len(kk), _p(out))
        return out


def threads() -> int:
    return int(os.environ.get("OMP_NUM_THREADS", len(os.sched_getaffinity(0))))
