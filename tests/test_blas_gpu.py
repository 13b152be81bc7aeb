"""Parity of the sm_100a BLAS kernels (vadd/vsub/vmul/axpy) with the oracle,
through the C ABI.  Bit-exact everywhere (integer work)."""

from __future__ import annotations

import hashlib
import random

import numpy as np
import pytest

from oracle import bigint
from oracle.cbind import OracleField

pytestmark = pytest.mark.gpu

WIDTHS = [16, 32, 64, 96, 128, 160, 192, 224, 256, 288, 320, 352, 384, 416, 448, 480, 512, 544, 640, 768, 800, 1024]


def _dev():
    from paper_2501_07535_b200 import device
    return device


def _native_limbs():
    import ctypes
    from paper_2501_07535_b200 import _lib
    buf = (ctypes.c_int * 64)()
    m = _lib.load().wm_supported_limbs(0, buf, 64)
    return set(buf[:m])


def run_op(kind, bits, q, xs, ys, scalar=0, strategy="schoolbook"):
    dev = _dev()
    f = dev.Field(bits, q, strategy)
    x = dev.to_device(dev.ints_to_limbs(xs, f.limbs))
    y = dev.to_device(dev.ints_to_limbs(ys, f.limbs))
    out = f.axpy(scalar, x, y) if kind == "axpy" else getattr(f, kind)(x, y)
    return dev.limbs_to_ints(dev.to_host(out))


def test_reference_pins(cuda):  # reference test_kernels.py:82-90,113-120 (q=500 is even)
    from paper_2501_07535_b200 import kernels as K
    from paper_2501_07535_b200.params import compute_barrett
    L13 = K.WordLayout(13, 8)
    Q500 = compute_barrett(500, 13)
    vadd = K.build_program(K.KernelSpec("vadd", L13, 4, Q500))
    assert K.run_vector(vadd, [300, 499, 0, 250], [400, 1, 0, 250]) == [200, 0, 0, 0]
    axpy = K.build_program(K.KernelSpec("axpy", L13, 3, Q500))
    assert K.run_vector(axpy, 0, [5, 6, 7], [9, 8, 7]) == [9, 8, 7]
    vmul = K.build_program(K.KernelSpec("vmul", L13, 3, Q500))
    assert K.run_vector(vmul, [1, 1, 1], [123, 456, 499]) == [123, 456, 499]
    assert K.run_program(K.build_program(K.KernelSpec("addmod", L13, 1, Q500)), 300, 400) == 200
    assert K.run_program(K.build_program(K.KernelSpec("submod", L13, 1, Q500)), 100, 300) == 300
    mul = K.build_program(K.make_spec("mulmod", 16, 8))
    assert K.run_program(mul, 3000, 2000) == 3755


def test_golden_vectors(cuda, golden):
    """Reference run_vector outputs (lowered reference kernels, make_golden.py)."""
    for row in golden("blas"):
        q = int(row["q"])
        xs = [int(v) for v in row["a"]]
        ys = [int(v) for v in row["b"]]
        got = run_op(row["kind"], row["bits"], q, xs, ys, int(row.get("scalar", 0)))
        assert got == [int(v) for v in row["out"]], (row["kind"], row["bits"])


@pytest.mark.parametrize("strategy", ["schoolbook", "karatsuba"])
def test_api_run_vector_matches_reference_goldens(cuda, golden, strategy):
    """Through the reference-mirroring API, incl. make_spec(strategy=...)
    (reference kernels.py:104-117)."""
    from paper_2501_07535_b200 import kernels as K
    for row in golden("blas"):
        spec = K.make_spec(row["kind"], row["bits"], row["word"], size=len(row["a"]), strategy=strategy)
        prog = K.generate_kernel(spec)
        xs = [int(v) for v in row["a"]]
        ys = [int(v) for v in row["b"]]
        args = (int(row["scalar"]), xs, ys) if row["kind"] == "axpy" else (xs, ys)
        assert K.run_vector(prog, *args) == [int(v) for v in row["out"]]


@pytest.mark.parametrize("bits", WIDTHS)
@pytest.mark.parametrize("kind", ["vadd", "vsub", "vmul", "axpy", "vmul_karatsuba", "axpy_karatsuba"])
def test_random_and_edges_vs_oracle(cuda, bits, kind):
    """Reference moduli (largest prime below 2^(bits-4)) and a random general
    modulus in the Barrett range; seeded inputs plus the {0,1,q-1}^2 grid."""
    from paper_2501_07535_b200.params import find_ntt_params
    rnd = random.Random(bits * 31 + len(kind))
    qs = [find_ntt_params(bits, 1).p,
          rnd.randrange((1 << (bits - 5)) + 1, 1 << (bits - 4)) | 1,
          rnd.randrange((1 << (bits - 5)) + 1, 1 << (bits - 4)) & ~1]
    for q in qs:
        n = 3000
        rng = np.random.Generator(np.random.PCG64(bits))
        xs = bigint.uniform_residues(rng, n, q)
        ys = bigint.uniform_residues(rng, n, q)
        edge = (0, 1, q - 1)
        xs += [a for a in edge for _ in edge]
        ys += [b for _ in edge for b in edge]
        s = rnd.randrange(q)
        op, _, strat = kind.partition("_")
        if q % 2 == 0 and (bits + 31) // 32 not in _native_limbs():
            # widths without kernels of their own run zero-padded Montgomery
            # fields, which need an odd modulus
            from paper_2501_07535_b200 import _lib
            with pytest.raises(_lib.Unsupported):
                run_op(op, bits, q, xs, ys, s, strat or "schoolbook")
            continue
        got = run_op(op, bits, q, xs, ys, s, strat or "schoolbook")
        kind = op
        if kind == "vadd":
            want = [(a + b) % q for a, b in zip(xs, ys)]
        elif kind == "vsub":
            want = [(a - b) % q for a, b in zip(xs, ys)]
        elif kind == "vmul":
            want = [a * b % q for a, b in zip(xs, ys)]
        else:
            want = [(s * a + b) % q for a, b in zip(xs, ys)]
        assert got == want, (kind, bits, q)


@pytest.mark.parametrize("strategy", ["schoolbook", "karatsuba"])
def test_adversarial_vmul_operands(cuda, strategy):
    """Operands that maximise the Barrett quotient error: q-1, q-2, values
    near powers of two, and all-ones limbs below q."""
    from paper_2501_07535_b200.params import find_ntt_params
    for bits in (64, 128, 256, 384, 512, 768, 1024):
        q = find_ntt_params(bits, 1).p
        specials = [q - 1, q - 2, (q - 1) // 2, (q + 1) // 2, 1 << (bits - 5), (1 << (bits - 5)) - 1,
                    q - (1 << 32), (1 << 32) - 1, 2, 3]
        xs = [a for a in specials for _ in specials]
        ys = [b for _ in specials for b in specials]
        assert run_op("vmul", bits, q, xs, ys, 0, strategy) == [a * b % q for a, b in zip(xs, ys)]


def test_aliasing_and_sizes(cuda):
    dev = _dev()
    import torch
    q = (1 << 252) - 129
    f = dev.Field(256, q)
    for n in (1, 7, 255, 256, 257, 100_003):
        rng = np.random.Generator(np.random.PCG64(n))
        xs = bigint.uniform_residues(rng, n, q)
        ys = bigint.uniform_residues(rng, n, q)
        x = dev.to_device(dev.ints_to_limbs(xs, 8))
        y = dev.to_device(dev.ints_to_limbs(ys, 8))
        f.vmul(x, y, out=x)  # out aliases a
        assert dev.limbs_to_ints(dev.to_host(x))[:50] == [a * b % q for a, b in zip(xs[:50], ys[:50])]
        assert dev.limbs_to_ints(dev.to_host(x))[-5:] == [a * b % q for a, b in zip(xs[-5:], ys[-5:])]
    empty = torch.empty((0, 8), dtype=torch.int32, device="cuda")
    assert f.vadd(empty, empty).numel() == 0
    with pytest.raises(ValueError):
        f.vadd(torch.zeros((4, 8), dtype=torch.int32, device="cuda"),
               torch.zeros((5, 8), dtype=torch.int32, device="cuda"))


@pytest.mark.parametrize("bits", [128, 256, 384, 768])
def test_full_size_checksum_vs_c_oracle(cuda, bits):
    """BASELINE config 3 sizes (n=2^24 at 128/256-bit, 2^22 above): device
    output checksum equals the C oracle's (reference Barrett semantics)."""
    from paper_2501_07535_b200.params import find_ntt_params
    dev = _dev()
    import torch
    n = 1 << 24 if bits <= 256 else 1 << 22
    q = find_ntt_params(bits, 1).p
    K = (bits + 31) // 32
    g = torch.Generator(device="cuda").manual_seed(bits)
    # canonical inputs: top limb masked to bits-5 bits (< 2^(bits-5) < q)
    x = torch.randint(-(1 << 31), 1 << 31, (n, K), dtype=torch.int32, device="cuda", generator=g)
    y = torch.randint(-(1 << 31), 1 << 31, (n, K), dtype=torch.int32, device="cuda", generator=g)
    top = (1 << (bits - 5 - 32 * (K - 1))) - 1
    x[:, K - 1] &= top
    y[:, K - 1] &= top
    f = dev.Field(bits, q)
    of = OracleField(q, bits)
    xh, yh = dev.to_host(x), dev.to_host(y)
    for kind in ("vmul", "axpy", "vadd"):
        out = f.axpy(12345, x, y) if kind == "axpy" else getattr(f, kind)(x, y)
        want = of.vector(kind, xh, yh, 12345)
        got = dev.to_host(out)
        assert hashlib.sha256(got.tobytes()).digest() == hashlib.sha256(want.tobytes()).digest(), (kind, bits)


def test_ref_layout_roundtrip(cuda):
    """Reference AoS MSW-first words (kernels.to_words) <-> device limbs."""
    dev = _dev()
    import torch
    from paper_2501_07535_b200 import kernels as K
    for bits, word in [(256, 64), (256, 32), (384, 64), (768, 32), (128, 64)]:
        lay = K.WordLayout(bits, word)
        q = (1 << (bits - 4)) - 1
        rnd = random.Random(bits)
        vals = [rnd.randrange(q) for _ in range(100)]
        flat = [w for v in vals for w in K.to_words(v, lay.padded_words, word)]
        dt = np.uint64 if word == 64 else np.uint32
        ref = torch.from_numpy(np.array(flat, dtype=dt).view(np.int64 if word == 64 else np.int32)).cuda()
        f = dev.Field(bits, find_prime_below(bits))
        limbs = f.from_ref_layout(ref, word, lay.padded_words)
        assert dev.limbs_to_ints(dev.to_host(limbs)) == vals
        back = f.to_ref_layout(limbs, word, lay.padded_words)
        assert torch.equal(back.view(-1), ref)


def find_prime_below(bits):
    from paper_2501_07535_b200.params import find_ntt_params
    return find_ntt_params(bits, 1).p


def test_widemul_full_products(cuda):
    """Bare widening multiply (reference build_wide_mul, kernels.py:314-329):
    test_kernels.py:266-269 pins plus random operands at several widths and
    both strategies."""
    from paper_2501_07535_b200 import kernels as K
    prog = K.generate_kernel(K.make_spec("widemul", 16, 8))
    assert K.run_program(prog, 0xFFFF, 0xFFFF) == 0xFFFF * 0xFFFF
    assert K.run_program(prog, 1234, 4321) == 1234 * 4321
    rnd = random.Random(5)
    for bits in (64, 256, 384, 640, 1024):
        for strat in ("schoolbook", "karatsuba"):
            wm = K.generate_kernel(K.make_spec("widemul", bits, 32, strategy=strat))
            xs = [rnd.getrandbits(bits) for _ in range(500)] + [(1 << bits) - 1, 0, 1]
            ys = [rnd.getrandbits(bits) for _ in range(500)] + [(1 << bits) - 1, (1 << bits) - 1, 1]
            assert K.run_vector(wm, xs, ys) == [a * b for a, b in zip(xs, ys)], (bits, strat)


@pytest.mark.parametrize("bits", [32, 64, 128])
@pytest.mark.parametrize("offset", [0, 1, 3])
def test_small_elements_packed_and_unaligned(cuda, bits, offset):
    """1-, 2- and 4-limb elements take packed 256-bit accesses (8/K elements
    per thread) when the three bases are 32-byte aligned, one element per
    thread otherwise; both paths and the ragged n % (8/K) tail must agree with
    Python integers.  Views at an element offset make the bases unaligned."""
    torch = cuda
    dev = _dev()
    rnd = random.Random(bits * 10 + offset)
    q = (1 << (bits - 4)) - 59 if bits > 32 else 4294967291 >> 4
    f = dev.Field(bits, q)
    n = 4099  # odd: every packing leaves a tail
    xs = [rnd.randrange(q) for _ in range(n + offset)]
    ys = [rnd.randrange(q) for _ in range(n + offset)]
    x = dev.to_device(dev.ints_to_limbs(xs, f.limbs))[offset:]
    y = dev.to_device(dev.ints_to_limbs(ys, f.limbs))[offset:]
    outbuf = torch.empty((n + offset, f.limbs), dtype=torch.int32, device="cuda")
    out = outbuf[offset:]
    a, b = xs[offset:], ys[offset:]
    s = rnd.randrange(q)
    for kind, want in (("vadd", [(u + v) % q for u, v in zip(a, b)]),
                       ("vsub", [(u - v) % q for u, v in zip(a, b)]),
                       ("vmul", [u * v % q for u, v in zip(a, b)]),
                       ("axpy", [(s * u + v) % q for u, v in zip(a, b)])):
        r = f.axpy(s, x, y, out=out) if kind == "axpy" else getattr(f, kind)(x, y, out=out)
        assert dev.limbs_to_ints(dev.to_host(r)) == want, (kind, bits, offset)


@pytest.mark.parametrize("bits,strategy,reduction", [(768, "karatsuba", "barrett"), (768, "schoolbook", "barrett"),
                                                     (1024, "karatsuba", "barrett"), (256, "schoolbook", "auto"),
                                                     (256, "karatsuba", "auto")])
def test_tma_staged_path(cuda, bits, strategy, reduction):
    """The TMA-staged kernel (generic Barrett vmul/axpy from 24 limbs, the
    256-bit special-form axpy): several tiles per CTA (stage reuse, both
    mbarrier phases), a ragged tail of n mod 256 elements, an element-offset
    view, and out aliasing an input, all against Python ints."""
    import torch
    dev = _dev()
    from paper_2501_07535_b200.params import find_ntt_params
    q = find_ntt_params(bits, 1).p
    f = dev.Field(bits, q, strategy, reduction=reduction)
    r = random.Random(bits)
    n = 256 * 700 + 77
    xs = [r.randrange(q) for _ in range(n + 1)]
    ys = [r.randrange(q) for _ in range(n)]
    ys[:3] = [0, 1, q - 1]
    xs[1:4] = [q - 1, q - 1, 0]
    xd = dev.to_device(dev.ints_to_limbs(xs, f.limbs))[1:]  # element-offset view
    yd = dev.to_device(dev.ints_to_limbs(ys, f.limbs))
    want = [a * b % q for a, b in zip(xs[1:], ys)]
    assert dev.limbs_to_ints(dev.to_host(f.vmul(xd, yd))) == want
    a = r.randrange(q)
    want_axpy = [(a * x + y) % q for x, y in zip(xs[1:], ys)]
    y2 = yd.clone()
    f.axpy(a, xd, y2, out=y2)  # out aliases y
    assert dev.limbs_to_ints(dev.to_host(y2)) == want_axpy
    torch.cuda.synchronize()
