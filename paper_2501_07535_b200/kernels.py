"""Operator API of the reference ``widemod.kernels``, executed on the B200.

Every public name here keeps the reference's signature, argument meaning and
error behaviour (reference pkg/src/widemod/kernels.py, cited per function),
so code written against ``widemod.kernels`` for the hot path — building a
spec, generating a kernel, ``run_vector`` / ``run_ntt`` — runs unchanged.
What changes is the execution: ``generate_kernel`` returns a handle to the
sm_100a kernels of ``libwidemod_b200.so`` (instead of a lowered straight-line
IR program) and the ``run_*`` executors move the operands to the GPU, launch,
and copy the results back.  There is no CPU execution path.

Out of scope (not on the hot path): the IR, the rewrite engine,
the C/CUDA text emitters and the front ends.  ``params_mode`` is accepted for
compatibility; the device kernels always take the modulus at run time.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from .device import Field, NttPlan, ints_to_limbs, limbs_for_bits, limbs_to_ints, to_device, to_host
from .params import BarrettParams, NttParams, compute_barrett, find_ntt_params

SCALAR_KINDS = ("addmod", "submod", "mulmod")
VECTOR_KINDS = ("vadd", "vsub", "vmul", "axpy")
NTT_KINDS = ("ntt", "intt")
KERNEL_KINDS = SCALAR_KINDS + VECTOR_KINDS + NTT_KINDS + ("widemul",)

PARAMS_MODES = ("baked", "runtime")

_SCALAR_TO_VECTOR = {"addmod": "vadd", "submod": "vsub", "mulmod": "vmul"}


class InvalidKernel(ValueError):
    """Kernel kind/size/parameter combination that cannot be built
    (reference kernels.py:36-37)."""


@dataclass(frozen=True)
class WordLayout:
    """Interface width on machine words (reference kernels.py:40-71).

    The device kernels always use 32-bit limbs (``limbs``); ``word_bits`` and
    the padded quantities describe the reference's AoS MSW-first word layout
    that ``wm_ref_to_limbs`` / ``wm_limbs_to_ref`` convert from/to."""

    bits: int
    word_bits: int

    def __post_init__(self) -> None:
        if self.word_bits not in (8, 16, 32, 64):
            raise InvalidKernel(f"word must be 8/16/32/64 bits, got {self.word_bits}")
        if self.bits < self.word_bits:
            raise InvalidKernel(f"interface width {self.bits} below word width {self.word_bits}")

    @property
    def words(self) -> int:
        return -(-self.bits // self.word_bits)

    @property
    def padded_words(self) -> int:
        return 1 << (self.words - 1).bit_length()

    @property
    def padded_bits(self) -> int:
        return self.padded_words * self.word_bits

    @property
    def limbs(self) -> int:
        """32-bit limbs per value in device memory (no power-of-two padding)."""
        return limbs_for_bits(self.bits)


@dataclass(frozen=True)
class KernelSpec:
    """Everything needed to rebuild a kernel (reference kernels.py:74-101)."""

    kind: str
    layout: WordLayout
    size: int = 1
    barrett: BarrettParams | None = None
    ntt: NttParams | None = None
    mul_strategy: str = "schoolbook"

    def __post_init__(self) -> None:
        if self.kind not in KERNEL_KINDS:
            raise InvalidKernel(f"unknown kernel kind {self.kind!r}")
        if self.kind in SCALAR_KINDS + ("widemul",) and self.size != 1:
            raise InvalidKernel(f"{self.kind} takes no size")
        if self.kind in VECTOR_KINDS and self.size < 1:
            raise InvalidKernel("vector size must be positive")
        if self.kind in NTT_KINDS:
            if self.ntt is None:
                raise InvalidKernel(f"{self.kind} needs transform parameters")
            if self.size != self.ntt.n:
                raise InvalidKernel("size disagrees with transform length")
        if self.kind != "widemul" and self.barrett is None:
            raise InvalidKernel(f"{self.kind} needs reduction parameters")
        if self.barrett is not None and self.barrett.width != self.layout.bits:
            raise InvalidKernel("reduction parameters built for a different width")


def make_spec(kind: str, bits: int, word: int, size: int = 1,
              strategy: str = "schoolbook") -> KernelSpec:
    """Pick the modulus (largest suitable prime) and assemble a spec
    (reference kernels.py:104-117)."""
    layout = WordLayout(bits, word)
    if kind == "widemul":
        return KernelSpec(kind, layout, 1, None, None, strategy)
    if kind in NTT_KINDS:
        params = find_ntt_params(bits, size)
        return KernelSpec(kind, layout, size, compute_barrett(params.p, bits), params, strategy)
    q = find_ntt_params(bits, 1).p
    n = size if kind in VECTOR_KINDS else 1
    return KernelSpec(kind, layout, n, compute_barrett(q, bits), None, strategy)


# ------------------------------------------------------------ device state
_cache_lock = threading.Lock()
_fields: dict = {}
_plans: dict = {}


def get_field(bits: int, q: int, strategy: str = "schoolbook") -> Field:
    """Shared device field for (width, modulus, multiplication strategy)."""
    key = (bits, q, strategy)
    with _cache_lock:
        f = _fields.get(key)
        if f is None:
            f = Field(bits, q, strategy)
            _fields[key] = f
        return f


def get_plan(bits: int, params: NttParams) -> NttPlan:
    """Shared device NTT plan for (width, transform parameters)."""
    key = (bits, params)
    field = get_field(bits, params.p)
    with _cache_lock:
        pl = _plans.get(key)
        if pl is None:
            pl = NttPlan(field, params)
            _plans[key] = pl
        return pl


class _Attrs(dict):
    """Program attributes; the twiddle list (n/2 big ints, as the reference
    stores it, kernels.py:300) is materialised only when asked for."""

    def __init__(self, *a, twiddle_source=None, **kw):
        super().__init__(*a, **kw)
        self._tw = twiddle_source

    def __missing__(self, key):
        if key == "twiddles" and self._tw is not None:
            params, inverse = self._tw
            val = [str(x) for x in twiddle_table(params, inverse)]
            self["twiddles"] = val
            return val
        raise KeyError(key)


class DeviceKernel:
    """What ``generate_kernel`` returns: a handle to the device kernels for a
    spec, carrying the reference Program's ``name`` and ``attributes``
    (kernels.py:156-165, 201-205, 244-249, 294-304) so executors and
    callers that read attributes keep working."""

    def __init__(self, spec: KernelSpec, params_mode: str = "baked"):
        if params_mode not in PARAMS_MODES:
            raise InvalidKernel(f"unknown params mode {params_mode!r}")
        self.spec = spec
        self.kind = spec.kind
        lay = spec.layout
        bp = spec.barrett
        if spec.kind == "widemul":  # bare widening multiply (kernels.py:314-329), no modulus
            self.name = f"widemul_{lay.bits}w{lay.word_bits}"
            self.attributes = _Attrs({
                "kernel": "widemul", "lambda": lay.bits, "omega0": lay.word_bits,
                "level_bits": lay.word_bits, "padded_bits": lay.padded_bits, "n": 1,
                "params_mode": params_mode, "limbs": lay.limbs, "arg_names": ["a", "b"],
                "ret_names": ["c"], "vector_args": [True, True]}, twiddle_source=None)
            return
        attrs = {
            "kernel": spec.kind,
            "lambda": lay.bits,
            "omega0": lay.word_bits,
            "level_bits": lay.word_bits,
            "padded_bits": lay.padded_bits,
            "n": 1,
            "params_mode": params_mode,
            "q": str(bp.q),
            "mu": str(bp.mu),
            "mbits": bp.mbits,
            "limbs": lay.limbs,
        }
        extra = ["q", "mu"] if params_mode == "runtime" else []
        tw_source = None
        if spec.kind in SCALAR_KINDS:
            self.name = f"{spec.kind}_{lay.bits}w{lay.word_bits}"
            extra = extra if spec.kind == "mulmod" else extra[:1]
            attrs.update(arg_names=["a", "b"] + extra, ret_names=["out"],
                         vector_args=[True, True] + [False] * len(extra))
        elif spec.kind in VECTOR_KINDS:
            self.name = f"{spec.kind}{spec.size}_{lay.bits}w{lay.word_bits}"
            extra = extra if spec.kind in ("vmul", "axpy") else extra[:1]
            args = ["a", "x", "y"] if spec.kind == "axpy" else ["a", "b"]
            vec = [False, True, True] if spec.kind == "axpy" else [True, True]
            attrs.update(n=spec.size, arg_names=args + extra, ret_names=["out"],
                         vector_args=vec + [False] * len(extra))
        else:
            nt = spec.ntt
            if nt.n < 2 or nt.n & (nt.n - 1):
                raise InvalidKernel(f"transform length {nt.n} is not a power of two at least 2")
            self.name = f"{spec.kind}{nt.n}_{lay.bits}w{lay.word_bits}"
            inverse = spec.kind == "intt"
            attrs.update(n=nt.n, p=str(nt.p), root=str(nt.root), root_inv=str(nt.root_inv),
                         n_inv=str(nt.n_inv), direction="inverse" if inverse else "forward",
                         arg_names=["u", "v", "w"] + extra, ret_names=["out0", "out1"])
            tw_source = (nt, inverse)
        self.attributes = _Attrs(attrs, twiddle_source=tw_source)

    @property
    def modulus(self) -> int:
        if self.spec.barrett is None:
            raise InvalidKernel(f"{self.kind} has no modulus")
        return self.spec.ntt.p if self.spec.ntt is not None else self.spec.barrett.q

    def field(self) -> Field:
        """Device field; the spec's mul_strategy ("schoolbook"/"karatsuba",
        reference KernelSpec.mul_strategy) selects the vmul/axpy multiplier."""
        _check_strategy(self.spec.mul_strategy)
        return get_field(self.spec.layout.bits, self.modulus, self.spec.mul_strategy)

    def plan(self) -> NttPlan:
        if self.spec.ntt is None:
            raise InvalidKernel(f"{self.kind} is not a transform")
        return get_plan(self.spec.layout.bits, self.spec.ntt)

    def __repr__(self) -> str:
        return f"DeviceKernel({self.name})"


def _check_strategy(strategy: str) -> None:
    """Reference RewriteConfig.__post_init__ (rewrite.py:55-56)."""
    if strategy not in ("schoolbook", "karatsuba"):
        raise ValueError(f"unknown strategy {strategy!r}")


def build_program(spec: KernelSpec, params_mode: str = "baked") -> DeviceKernel:
    """Reference kernels.py:332-340; returns the device kernel handle."""
    return DeviceKernel(spec, params_mode)


def _check_params_mode(params_mode: str) -> None:
    if params_mode not in PARAMS_MODES:
        raise InvalidKernel(f"unknown params mode {params_mode!r}")


def build_scalar(kind: str, layout: WordLayout, barrett: BarrettParams,
                 params_mode: str = "baked") -> DeviceKernel:
    """addmod / submod / mulmod on one element (reference kernels.py:184-212).
    ``run_program`` executes it on the device."""
    if kind not in SCALAR_KINDS:
        raise InvalidKernel(f"not a scalar kernel: {kind!r}")
    _check_params_mode(params_mode)
    return DeviceKernel(KernelSpec(kind, layout, 1, barrett), params_mode)


def build_vector(kind: str, layout: WordLayout, size: int, barrett: BarrettParams,
                 params_mode: str = "baked") -> DeviceKernel:
    """Elementwise vadd / vsub / vmul / axpy over ``size`` elements (reference
    kernels.py:215-256); ``run_vector`` executes it on the device."""
    if kind not in VECTOR_KINDS:
        raise InvalidKernel(f"not a vector kernel: {kind!r}")
    if size < 1:
        raise InvalidKernel("vector size must be positive")
    _check_params_mode(params_mode)
    return DeviceKernel(KernelSpec(kind, layout, size, barrett), params_mode)


def build_ntt(kind: str, layout: WordLayout, params: NttParams,
              params_mode: str = "baked") -> DeviceKernel:
    """Forward / inverse transform over ``params`` (reference kernels.py:270-311;
    the reference builds one butterfly plus schedule data, the device handle
    runs whole transforms through ``run_ntt`` and single butterflies through
    ``run_program``)."""
    if kind not in NTT_KINDS:
        raise InvalidKernel(f"not a transform kernel: {kind!r}")
    _check_params_mode(params_mode)
    if params.n < 2 or params.n & (params.n - 1):
        raise InvalidKernel(f"transform length {params.n} is not a power of two at least 2")
    barrett = compute_barrett(params.p, layout.bits)
    return DeviceKernel(KernelSpec(kind, layout, params.n, barrett, params), params_mode)


def build_wide_mul(layout: WordLayout) -> DeviceKernel:
    """Bare widening multiply a * b -> 2 x width (reference kernels.py:314-329)."""
    return DeviceKernel(KernelSpec("widemul", layout), "baked")


def generate_kernel(spec: KernelSpec, params_mode: str = "baked", target_has_double_word: bool = True,
                    prune: bool = True, trace: list | None = None) -> DeviceKernel:
    """Reference kernels.py:368-381.  The lowering/pruning the reference does
    here is compile-time template unrolling of the device library, so the
    flags are accepted and have no effect; ``trace`` receives one line."""
    # reference: RewriteConfig(mul_strategy=...) raises for an unknown strategy (rewrite.py:55-56)
    _check_strategy(spec.mul_strategy)
    kern = DeviceKernel(spec, params_mode)
    if trace is not None:
        trace.append(f"device {kern.name}: {spec.layout.limbs} x 32-bit limbs (sm_100a)")
    return kern


# ------------------------------------------------------------ schedules
def twiddle_table(params: NttParams, inverse: bool = False) -> list[int]:
    """Powers of root (root_inv), length n/2 (reference kernels.py:259-267)."""
    base = params.root_inv if inverse else params.root
    out = [1]
    for _ in range(max(1, params.n // 2) - 1):
        out.append(out[-1] * base % params.p)
    return out


def bit_reverse_order(n: int) -> list[int]:
    """Reference kernels.py:386-392."""
    if n & (n - 1) or n < 1:
        raise InvalidKernel(f"length {n} is not a power of two")
    bits = n.bit_length() - 1
    if bits == 0:
        return [0]
    idx = np.arange(n, dtype=np.int64)
    rev = np.zeros(n, dtype=np.int64)
    for b in range(bits):
        rev |= ((idx >> b) & 1) << (bits - 1 - b)
    return rev.tolist()


def butterfly_schedule(n: int) -> list[tuple[int, int, int]]:
    """(top, bottom, twiddle exponent) triples, stages m = 2..n
    (reference kernels.py:395-413)."""
    if n & (n - 1) or n < 2:
        raise InvalidKernel(f"length {n} is not a power of two at least 2")
    out = []
    m = 2
    while m <= n:
        half, step = m // 2, n // m
        for base in range(0, n, m):
            out.extend((base + j, base + j + half, j * step) for j in range(half))
        m *= 2
    return out


def to_words(value: int, count: int, width: int) -> list[int]:
    """MSW-first word split (reference kernels.py:418-421)."""
    mask = (1 << width) - 1
    return [(value >> (width * (count - 1 - i))) & mask for i in range(count)]


def from_words(words, width: int) -> int:
    """Reference kernels.py:424-428."""
    acc = 0
    for w in words:
        acc = (acc << width) | w
    return acc


# ------------------------------------------------------------ executors
def _check_canonical(values, bound: int, what: str) -> None:
    for v in values:
        if not 0 <= v < bound:
            raise ValueError(f"{what} operand {v} is not a canonical residue mod {bound}")


def _vector_launch(kern: DeviceKernel, op: str, arrays) -> list[int]:
    field = kern.field()
    K = field.limbs
    if op == "axpy":
        a, xs, ys = arrays
        _check_canonical([a], field.q, "axpy scalar")
        _check_canonical(xs, field.q, "axpy x")
        _check_canonical(ys, field.q, "axpy y")
        x = to_device(ints_to_limbs(xs, K))
        y = to_device(ints_to_limbs(ys, K))
        out = field.axpy(a, x, y)
    else:
        xs, ys = arrays
        _check_canonical(xs, field.q, op)
        _check_canonical(ys, field.q, op)
        x = to_device(ints_to_limbs(xs, K))
        y = to_device(ints_to_limbs(ys, K))
        out = getattr(field, op)(x, y)
    return limbs_to_ints(to_host(out))


def _widemul_launch(kern: DeviceKernel, xs, ys) -> list[int]:
    """Full products a*b on the device (C ABI wm_widemul); operands are
    unsigned values below 2^(32 * storage limbs)."""
    from . import _lib
    from .device import _stream_ptr, _torch
    torch = _torch()
    bits = kern.spec.layout.bits
    lib = _lib.load()
    K = lib.wm_limbs_for_bits(bits)
    if K < 1:
        raise _lib.Unsupported(f"width {bits} not built")
    for v in list(xs) + list(ys):
        if not 0 <= v < (1 << (32 * K)):
            raise ValueError(f"widemul operand {v} does not fit {bits} bits")
    x = to_device(ints_to_limbs(xs, K))
    y = to_device(ints_to_limbs(ys, K))
    out = torch.empty((len(xs), 2 * K), dtype=torch.int32, device="cuda")
    _lib.check(lib.wm_widemul(bits, 1 if kern.spec.mul_strategy == "karatsuba" else 0, x.data_ptr(),
                              y.data_ptr(), out.data_ptr(), len(xs), _stream_ptr(None)), "wm_widemul")
    return limbs_to_ints(to_host(out))


def run_program(program: DeviceKernel, *args, fn=None):
    """Run a kernel on single operands (reference kernels.py:442-464).
    Scalar kinds take (a, b); vector kinds take one element per argument;
    transforms take (u, v, w) and return the butterfly (u + v*w, u - v*w)."""
    kind = program.kind
    if kind == "widemul":
        if len(args) != 2:
            raise TypeError(f"{len(args)} operands for 2 parameters")
        return _widemul_launch(program, [args[0]], [args[1]])[0]
    if kind in SCALAR_KINDS or kind in ("vadd", "vsub", "vmul"):
        if len(args) != 2:
            raise TypeError(f"{len(args)} operands for 2 parameters")
        op = _SCALAR_TO_VECTOR.get(kind, kind)
        return _vector_launch(program, op, ([args[0]], [args[1]]))[0]
    if kind == "axpy":
        if len(args) != 3:
            raise TypeError(f"{len(args)} operands for 3 parameters")
        return _vector_launch(program, "axpy", (args[0], [args[1]], [args[2]]))[0]
    if len(args) != 3:
        raise TypeError(f"{len(args)} operands for 3 parameters")
    u, v, w = args
    p = program.spec.ntt.p
    field = get_field(program.spec.layout.bits, p)
    K = field.limbs
    _check_canonical([u, v, w], p, "butterfly")
    t = field.vmul(to_device(ints_to_limbs([v], K)), to_device(ints_to_limbs([w], K)))
    ud = to_device(ints_to_limbs([u], K))
    o0 = limbs_to_ints(to_host(field.vadd(ud, t)))[0]
    o1 = limbs_to_ints(to_host(field.vsub(ud, t)))[0]
    return o0, o1


def run_vector(program: DeviceKernel, *arrays, fn=None) -> list[int]:
    """Element-wise kernel over whole vectors (reference kernels.py:467-480):
    arrays are (a, b) for vadd/vsub/vmul and (a_scalar, x, y) for axpy;
    ValueError on a length mismatch."""
    attrs = program.attributes
    if program.kind == "widemul":  # the reference maps run_program over the elements
        if len(arrays) != 2:
            raise TypeError(f"{len(arrays)} operands for 2 parameters")
        if len(arrays[0]) != len(arrays[1]):
            raise ValueError(f"expected {len(arrays[0])} elements, got {len(arrays[1])}")
        return _widemul_launch(program, arrays[0], arrays[1])
    if program.kind not in VECTOR_KINDS:
        raise InvalidKernel(f"{program.kind} is not a vector kernel")
    n = attrs["n"]
    flags = attrs["vector_args"][:len(arrays)]
    for arr, is_vec in zip(arrays, flags):
        if is_vec and len(arr) != n:
            raise ValueError(f"expected {n} elements, got {len(arr)}")
    want = 3 if program.kind == "axpy" else 2
    if len(arrays) != want:
        raise TypeError(f"{len(arrays)} operands for {want} parameters")
    return _vector_launch(program, program.kind, arrays)


def run_ntt(program: DeviceKernel, values, fn=None) -> list[int]:
    """Full transform, natural order in and out (reference kernels.py:483-499)."""
    attrs = program.attributes
    if program.kind not in NTT_KINDS:
        raise InvalidKernel(f"{program.kind} is not a transform")
    n = attrs["n"]
    if len(values) != n:
        raise ValueError(f"expected {n} elements, got {len(values)}")
    return run_ntt_batch(program, [values])[0]


def run_ntt_batch(program: DeviceKernel, vectors) -> list[list[int]]:
    """Batched ``run_ntt``: one device launch sequence for all vectors."""
    plan = program.plan()
    n = plan.n
    p = program.spec.ntt.p
    flat = []
    for vec in vectors:
        if len(vec) != n:
            raise ValueError(f"expected {n} elements, got {len(vec)}")
        _check_canonical(vec, p, program.kind)
        flat.extend(vec)
    if not flat:
        return []
    x = to_device(ints_to_limbs(flat, plan.limbs))
    y = plan.inverse(x) if program.kind == "intt" else plan.forward(x)
    out = limbs_to_ints(to_host(y))
    return [out[i * n:(i + 1) * n] for i in range(len(vectors))]
