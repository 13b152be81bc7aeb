"""Device-resident objects over the C ABI: fields, NTT plans, limb tensors.

Data live in CUDA memory as ``torch.int32`` tensors of shape ``[..., K]``
holding the uint32 limbs of each value, least-significant limb first and
element after element (the layout of include/widemod_b200.h).  PyTorch is
only the allocator/stream provider here; every arithmetic operation is a
kernel in ``libwidemod_b200.so``.  There is no CPU fallback: without a CUDA
device or without the library every method raises.
"""

from __future__ import annotations

import ctypes
from typing import Iterable, Sequence

import numpy as np

from . import _lib
from .params import NttParams

_i = ctypes.c_int


def limbs_for_bits(bits: int) -> int:
    """32-bit limbs per value of an interface width (ceil(bits/32))."""
    if bits < 1:
        raise ValueError(f"bad width {bits}")
    return (bits + 31) // 32


try:  # C loop over the interpreter's int <-> bytes conversions (csrc/host/wm_conv.c)
    from . import _wmconv
except ImportError:  # not built on this host: the same conversion per element in Python
    _wmconv = None


def ints_to_limbs(values: Iterable[int], limbs: int) -> np.ndarray:
    """Python ints -> uint32 array [len, limbs], little-endian limbs
    (reference to_words, kernels.py:418-421, without the MSW-first order)."""
    nbytes = 4 * limbs
    try:
        if _wmconv is not None:
            vals = values if isinstance(values, (list, tuple)) else list(values)
            buf = _wmconv.ints_to_limbs(vals, limbs)
        else:
            buf = b"".join(int(v).to_bytes(nbytes, "little") for v in values)
    except OverflowError as exc:
        raise ValueError(f"value does not fit in {limbs} limbs (or is negative)") from exc
    return np.frombuffer(buf, dtype="<u4").reshape(-1, limbs).copy()


def limbs_to_ints(arr: np.ndarray) -> list[int]:
    """uint32 array [len, limbs] -> Python ints (reference from_words)."""
    a = np.ascontiguousarray(arr, dtype="<u4")
    limbs = a.shape[-1]
    if _wmconv is not None:
        return _wmconv.limbs_to_ints(a.reshape(-1), limbs)
    raw = a.tobytes()
    step = 4 * limbs
    return [int.from_bytes(raw[i:i + step], "little") for i in range(0, len(raw), step)]


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise _lib.LibraryUnavailable("no CUDA device: the widemod_b200 kernels need a B200")
    return torch


def _stream_ptr(stream=None) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def to_device(arr: np.ndarray, device=None):
    """uint32 numpy limbs -> int32 CUDA tensor (same bits)."""
    torch = _torch()
    t = torch.from_numpy(np.ascontiguousarray(arr, dtype="<u4").view(np.int32))
    return t.to(device or "cuda", non_blocking=False)


def to_host(t) -> np.ndarray:
    """int32 CUDA tensor -> uint32 numpy limbs."""
    return t.detach().cpu().numpy().view("<u4")


def _ptr(t) -> int:
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()


class Field:
    """A modulus q at an interface width, with device reduction constants
    (C ABI ``wm_field_*``).  Replaces the baked q/mu of a generated reference
    kernel (kernels._param_vars, kernels.py:168-181)."""

    def __init__(self, bits: int, q: int, strategy: str = "schoolbook", reduction: str = "auto"):
        """strategy: full-product algorithm ("schoolbook"/"karatsuba") or a
        full-width modulus ("montgomery").  reduction: "auto" reduces products
        modulo a special-form q = 2^m - c (c < 2^32; every find_ntt_params
        modulus) by two folds and any other q by Barrett; "barrett" forces the
        generic Barrett path (WM_FIELD_BARRETT).  Results are identical."""
        self.lib = _lib.load()
        self.bits = int(bits)
        self.q = int(q)
        if strategy not in ("schoolbook", "karatsuba", "montgomery"):
            raise ValueError(f"unknown multiplication strategy {strategy!r}")
        if reduction not in ("auto", "barrett"):
            raise ValueError(f"unknown reduction {reduction!r}")
        self.strategy = strategy
        self.limbs = limbs_for_bits(self.bits)
        if self.q <= 1:
            raise ValueError(f"modulus must exceed 1, got {q}")
        ql = ints_to_limbs([self.q], self.limbs)[0]
        arr = _lib.u32_array(ql.tolist())
        h = ctypes.c_void_p()
        # "montgomery": full-width modulus (any odd q < 2^bits), Montgomery
        # products (the paper's full-width mode)
        flags = {"schoolbook": 0, "karatsuba": _lib.WM_FIELD_KARATSUBA,
                 "montgomery": _lib.WM_FIELD_MONTGOMERY}[strategy]
        if reduction == "barrett":
            flags |= _lib.WM_FIELD_BARRETT
        _lib.check(self.lib.wm_field_create_ex(self.bits, arr, self.limbs, flags, ctypes.byref(h)),
                   "wm_field_create_ex")
        self._h = h
        b, k, s = _i(), _i(), _i()
        _lib.check(self.lib.wm_field_info(self._h, ctypes.byref(b), ctypes.byref(k), ctypes.byref(s)))
        self.norm_shift = s.value
        red = self.lib.wm_field_reduction(self._h)
        if red < 0:
            _lib.check(-red, "wm_field_reduction")
        # the reduction the products use: "barrett", "montgomery" or "special_form"
        self.reduction = _lib.REDUCTION_NAMES[red]
        # storage limbs: ceil(bits/32), or the zero-padded limb count of a
        # width without kernels of its own (run as a Montgomery field)
        self.limbs = k.value

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self.lib.wm_field_destroy(h)
            except Exception:
                pass
            self._h = None

    # ---------------------------------------------------------------- BLAS
    def _check_vec(self, *ts):
        n = None
        for t in ts:
            if t.dtype.itemsize != 4 or t.shape[-1] != self.limbs:
                raise ValueError(f"expected int32 limbs [..., {self.limbs}]")
            m = t.numel() // self.limbs
            if n is None:
                n = m
            elif m != n:
                raise ValueError(f"expected {n} elements, got {m}")
        return n

    def _binop(self, fn, a, b, out, stream):
        torch = _torch()
        n = self._check_vec(a, b)
        if out is None:
            out = torch.empty_like(a)
        else:
            self._check_vec(a, out)
        _lib.check(fn(self._h, _ptr(a), _ptr(b), _ptr(out), n, _stream_ptr(stream)))
        return out

    def vadd(self, a, b, out=None, stream=None):
        """out = a + b mod q (reference vadd, kernels.py:235-236)."""
        return self._binop(self.lib.wm_vadd, a, b, out, stream)

    def vsub(self, a, b, out=None, stream=None):
        """out = a - b mod q (reference vsub, kernels.py:237-238)."""
        return self._binop(self.lib.wm_vsub, a, b, out, stream)

    def vmul(self, a, b, out=None, stream=None):
        """out = a * b mod q (reference vmul, kernels.py:239-240)."""
        return self._binop(self.lib.wm_vmul, a, b, out, stream)

    def axpy(self, a: int, x, y, out=None, stream=None):
        """out = a*x + y mod q for scalar a (reference axpy, kernels.py:241-243)."""
        torch = _torch()
        n = self._check_vec(x, y)
        if out is None:
            out = torch.empty_like(x)
        else:
            self._check_vec(x, out)
        if not 0 <= int(a) < self.q:
            raise ValueError("axpy scalar must be a canonical residue (0 <= a < q)")
        sl = _lib.u32_array(ints_to_limbs([int(a)], self.limbs)[0].tolist())
        _lib.check(self.lib.wm_axpy(self._h, sl, _ptr(x), _ptr(y), _ptr(out), n, _stream_ptr(stream)))
        return out

    def host_op(self, kind: str, a_host, b_host, out_host, scalar: int = 0, word_bits: int = 64,
                ref_words: int | None = None, chunk: int = 0, stream=None):
        """End-to-end BLAS on HOST tensors in the reference layout (AoS,
        MSW-first words, kernels.to_words): out = a (+,-,*) b, or
        out = scalar*a + b for "axpy", through the pipelined C ABI call
        ``wm_blas_host`` (chunked H2D / convert + kernel + convert / D2H on
        overlapping streams).  Pinned host tensors give full PCIe overlap."""
        codes = {"vadd": _lib.WM_OP_VADD, "vsub": _lib.WM_OP_VSUB, "vmul": _lib.WM_OP_VMUL,
                 "axpy": _lib.WM_OP_AXPY}
        if kind not in codes:
            raise ValueError(f"bad kind {kind!r}")
        if ref_words is None:
            ref_words = -(-self.bits // word_bits)
            ref_words = 1 << (ref_words - 1).bit_length()  # reference pads to a power of two
        per = ref_words * word_bits // 8
        for t in (a_host, b_host, out_host):
            if t.is_cuda or not t.is_contiguous():
                raise ValueError("host_op takes contiguous host tensors")
        nbytes = a_host.numel() * a_host.element_size()
        if nbytes % per or any(t.numel() * t.element_size() != nbytes for t in (b_host, out_host)):
            raise ValueError("host buffers differ in size or are not whole elements")
        sl = None
        if kind == "axpy":
            if not 0 <= int(scalar) < self.q:
                raise ValueError("axpy scalar must be a canonical residue (0 <= a < q)")
            sl = _lib.u32_array(ints_to_limbs([int(scalar)], self.limbs)[0].tolist())
        _lib.check(self.lib.wm_blas_host(self._h, codes[kind], sl, word_bits, ref_words, a_host.data_ptr(),
                                         b_host.data_ptr(), out_host.data_ptr(), nbytes // per, chunk,
                                         _stream_ptr(stream)), "wm_blas_host")
        return out_host

    def work(self, kind: str) -> float:
        """Word products one element of `kind` executes in this field's
        arithmetic (wm_blas_work): the executed-work basis of the BLAS
        integer roofline."""
        codes = {"vadd": _lib.WM_OP_VADD, "vsub": _lib.WM_OP_VSUB, "vmul": _lib.WM_OP_VMUL,
                 "axpy": _lib.WM_OP_AXPY}
        if kind not in codes:
            raise ValueError(f"bad kind {kind!r}")
        wp = ctypes.c_double()
        _lib.check(self.lib.wm_blas_work(self._h, codes[kind], ctypes.byref(wp)), "wm_blas_work")
        return wp.value

    # ---------------------------------------------------------------- layout
    def from_ref_layout(self, ref, word_bits: int, ref_words: int, out=None, stream=None):
        """Reference AoS MSW-first words (kernels.to_words) -> limb tensor."""
        torch = _torch()
        n = ref.numel() * ref.element_size() // (ref_words * word_bits // 8)
        if out is None:
            out = torch.empty((n, self.limbs), dtype=torch.int32, device=ref.device)
        _lib.check(self.lib.wm_ref_to_limbs(word_bits, ref_words, self.limbs, _ptr(ref), _ptr(out), n,
                                            _stream_ptr(stream)))
        return out

    def to_ref_layout(self, limbs_t, word_bits: int, ref_words: int, out=None, stream=None):
        """Limb tensor -> reference AoS MSW-first words."""
        torch = _torch()
        n = limbs_t.numel() // self.limbs
        if out is None:
            dt = torch.int64 if word_bits == 64 else torch.int32
            out = torch.empty((n, ref_words), dtype=dt, device=limbs_t.device)
        _lib.check(self.lib.wm_limbs_to_ref(word_bits, ref_words, self.limbs, _ptr(limbs_t), _ptr(out), n,
                                            _stream_ptr(stream)))
        return out


def probe_imad_wide(mode: int = 0, iters: int = 4096, stream=None) -> tuple[float, int]:
    """Measured 32x32->64 word-product throughput of this GPU (products/s)
    from wm_probe_imad_wide, timed with CUDA events; returns (rate, products)."""
    torch = _torch()
    lib = _lib.load()
    sink = torch.zeros(1, dtype=torch.int64, device="cuda")
    s = stream if stream is not None else torch.cuda.current_stream()
    prods = ctypes.c_int64()
    for _ in range(2):  # warm-up
        _lib.check(lib.wm_probe_imad_wide(mode, iters, sink.data_ptr(), int(s.cuda_stream), ctypes.byref(prods)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = None
    for _ in range(5):
        e0.record(s)
        _lib.check(lib.wm_probe_imad_wide(mode, iters, sink.data_ptr(), int(s.cuda_stream), ctypes.byref(prods)))
        e1.record(s)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return prods.value / (best * 1e-3), prods.value


class NttPlan:
    """Length-n NTT/INTT plan over a field's prime (C ABI ``wm_ntt_*``).

    Replaces the stage-per-launch transform of reference emit_cuda
    (emit.py:487-560) and the butterfly replay of run_ntt (kernels.py:483-499).
    Twiddle tables are generated on the device at construction."""

    def __init__(self, field: Field, params: NttParams):
        self.lib = field.lib
        self.field = field
        self.params = params
        self.n = int(params.n)
        if params.p != field.q:
            raise ValueError("transform prime differs from the field modulus")
        K = field.limbs
        enc = lambda v: _lib.u32_array(ints_to_limbs([v], K)[0].tolist())  # noqa: E731
        h = ctypes.c_void_p()
        _lib.check(self.lib.wm_ntt_plan_create(field.handle, self.n, enc(params.root), enc(params.root_inv),
                                               enc(params.n_inv), ctypes.byref(h)), "wm_ntt_plan_create")
        self._h = h
        npass = _i()
        sizes = (_i * 8)()
        _lib.check(self.lib.wm_ntt_plan_info(self._h, ctypes.byref(npass), sizes, 8))
        self.pass_log_sizes = [sizes[i] for i in range(npass.value)]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self.lib.wm_ntt_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def limbs(self) -> int:
        return self.field.limbs

    def workspace_bytes(self, batch: int) -> int:
        return int(self.lib.wm_ntt_workspace_bytes(self._h, batch))

    def _run(self, fn, x, out, workspace, stream):
        torch = _torch()
        K = self.limbs
        if x.dtype.itemsize != 4 or x.shape[-1] != K:
            raise ValueError(f"expected int32 limbs [..., {self.n}, {K}]")
        total = x.numel() // K
        if total % self.n:
            raise ValueError(f"expected a multiple of {self.n} elements, got {total}")
        batch = total // self.n
        if out is None:
            out = torch.empty_like(x)
        elif out.numel() != x.numel():
            raise ValueError("output size mismatch")
        ws = 0
        if workspace is not None:
            if workspace.numel() * workspace.element_size() < self.workspace_bytes(batch):
                raise ValueError("workspace too small")
            ws = _ptr(workspace)
        _lib.check(fn(self._h, _ptr(x), _ptr(out), batch, ws or None, _stream_ptr(stream)))
        return out

    def forward(self, x, out=None, workspace=None, stream=None):
        """y[k] = sum_j x[j] root^(jk) mod p per transform, natural order."""
        return self._run(self.lib.wm_ntt_forward, x, out, workspace, stream)

    def inverse(self, x, out=None, workspace=None, stream=None):
        """x[j] = n^-1 sum_k y[k] root^(-jk) mod p per transform."""
        return self._run(self.lib.wm_ntt_inverse, x, out, workspace, stream)

    def convolve(self, a, b, out=None, workspace=None, stream=None):
        """Cyclic convolution per transform: INTT(NTT(a) * NTT(b)) with the
        pointwise product fused into the forward transform of b."""
        torch = _torch()
        K = self.limbs
        for t in (a, b):
            if t.dtype.itemsize != 4 or t.shape[-1] != K:
                raise ValueError(f"expected int32 limbs [..., {self.n}, {K}]")
        if a.numel() != b.numel():
            raise ValueError("a and b differ in size")
        if out is None:
            out = torch.empty_like(a)
        elif out.numel() != a.numel() or out.dtype.itemsize != 4:
            raise ValueError("output size mismatch")
        if out.data_ptr() == b.data_ptr():
            raise ValueError("b may not alias out")
        total = a.numel() // K
        if total % self.n:
            raise ValueError(f"expected a multiple of {self.n} elements")
        batch = total // self.n
        ws = None
        if workspace is not None:
            if workspace.numel() * workspace.element_size() < self.workspace_bytes(batch):
                raise ValueError("workspace too small")
            ws = _ptr(workspace)
        _lib.check(self.lib.wm_ntt_convolve(self._h, _ptr(a), _ptr(b), _ptr(out), batch, ws, _stream_ptr(stream)),
                   "wm_ntt_convolve")
        return out

    def run_pass(self, pass_index: int, x, out, inverse: bool = False, stream=None):
        """Diagnostic: one pass kernel alone (wm_ntt_pass), for timing."""
        batch = x.numel() // (self.limbs * self.n)
        _lib.check(self.lib.wm_ntt_pass(self._h, 1 if inverse else 0, pass_index, _ptr(x), _ptr(out), batch,
                                        _stream_ptr(stream)), "wm_ntt_pass")
        return out

    def pass_work(self, pass_index: int, batch: int, inverse: bool = False) -> tuple[int, float]:
        """(field multiplications, word products) one pass kernel executes
        for `batch` transforms (wm_ntt_pass_work): the executed-work basis of
        the NTT roofline."""
        muls = ctypes.c_int64()
        wp = ctypes.c_double()
        _lib.check(self.lib.wm_ntt_pass_work(self._h, 1 if inverse else 0, pass_index, batch, ctypes.byref(muls),
                                             ctypes.byref(wp)), "wm_ntt_pass_work")
        return muls.value, wp.value

    def host_transform(self, host_in, host_out, mode: str = "forward", word_bits: int = 64,
                       ref_words: int | None = None, chunk: int = 0, stream=None):
        """End-to-end transform of HOST tensors in the reference layout (AoS,
        MSW-first words, kernels.to_words) through the pipelined C ABI call
        ``wm_ntt_host``: chunked H2D / kernels / D2H overlap.  mode is
        "forward", "inverse" or "forward_inverse" ("copy": the same pipeline
        without the transform, i.e. the PCIe floor of the call).  Pinned host tensors give
        full PCIe overlap."""
        codes = {"forward": _lib.WM_NTT_FWD, "inverse": _lib.WM_NTT_INV,
                 "forward_inverse": _lib.WM_NTT_FWD_INV, "copy": _lib.WM_NTT_COPY}
        if mode not in codes:
            raise ValueError(f"bad mode {mode!r}")
        if ref_words is None:
            ref_words = -(-self.field.bits // word_bits)
            ref_words = 1 << (ref_words - 1).bit_length()  # reference pads to a power of two
        if host_in.is_cuda or host_out.is_cuda:
            raise ValueError("host_transform takes host tensors")
        per = self.n * ref_words * word_bits // 8
        nbytes = host_in.numel() * host_in.element_size()
        if nbytes % per or host_out.numel() * host_out.element_size() != nbytes:
            raise ValueError("host buffers are not a whole number of transforms")
        if not (host_in.is_contiguous() and host_out.is_contiguous()):
            raise ValueError("expected contiguous host tensors")
        batch = nbytes // per
        if not (host_in.is_pinned() and host_out.is_pinned()):
            import warnings
            warnings.warn("host_transform with pageable host memory: copies cannot overlap (pin the buffers)",
                          RuntimeWarning, stacklevel=2)
        _lib.check(self.lib.wm_ntt_host(self._h, codes[mode], word_bits, ref_words, host_in.data_ptr(),
                                        host_out.data_ptr(), batch, chunk, _stream_ptr(stream)), "wm_ntt_host")
        return host_out

    def twiddles(self, count: int | None = None, inverse: bool = False, stream=None):
        """Device-generated powers root^e (root_inv^e), e < count."""
        torch = _torch()
        count = self.n // 2 if count is None else int(count)
        out = torch.empty((count, self.limbs), dtype=torch.int32, device="cuda")
        _lib.check(self.lib.wm_ntt_twiddles(self._h, 1 if inverse else 0, count, _ptr(out),
                                            _stream_ptr(stream)))
        return out
