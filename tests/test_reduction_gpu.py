"""Special-form (two-fold) reduction against the generic Barrett path and
Python big integers.

Every modulus the reference's find_ntt_params returns is q = 2^m - c with a
one-limb c (oracle.py:186-239: the largest primes below 2^(bits-4)), so the
library reduces those products by two folds (wm_limb.cuh mul_pm_lazy) unless
the field is created with reduction="barrett" (WM_FIELD_BARRETT).  Both must
give the reference's canonical residues bit for bit (reference
barrett_mulmod oracle.py:137-149; _emit_mulmod kernels.py:140-153)."""

from __future__ import annotations

import random

import numpy as np
import pytest

from oracle import bigint
from oracle.cbind import OracleField

pytestmark = pytest.mark.gpu


def _dev():
    from paper_2501_07535_b200 import device
    return device


def _operands(rng, q, n):
    xs = [rng.randrange(q) for _ in range(n)]
    ys = [rng.randrange(q) for _ in range(n)]
    edge = [0, 1, 2, q - 2, q - 1, q // 2, (1 << (q.bit_length() - 1)) - 1]
    edge = [e % q for e in edge]
    for a in edge:
        for b in edge:
            xs.append(a)
            ys.append(b)
    return xs, ys


def _run(field, kind, xs, ys, scalar=0):
    dev = _dev()
    x = dev.to_device(dev.ints_to_limbs(xs, field.limbs))
    y = dev.to_device(dev.ints_to_limbs(ys, field.limbs))
    out = field.axpy(scalar, x, y) if kind == "axpy" else getattr(field, kind)(x, y)
    return dev.limbs_to_ints(dev.to_host(out))


# (bits, m, c): q = 2^m - c.  The reference's BLAS moduli (m = bits - 4) plus
# the extremes of the special-form range (c = 1, c = 2^32 - 1, 32K - m = 4..31).
SPECIAL = [
    (128, 124, 59), (256, 252, 129), (384, 380, 65), (768, 764, 393),
    (96, 92, 1), (96, 72, (1 << 32) - 1), (160, 156, (1 << 32) - 1), (256, 225, 12345),
    (256, 252, (1 << 32) - 1), (512, 490, 3), (1024, 1020, 1 << 31), (320, 296, 77),
]


@pytest.mark.parametrize("bits,m,c", SPECIAL)
@pytest.mark.parametrize("strategy", ["schoolbook", "karatsuba"])
def test_special_form_matches_python_ints(cuda, bits, m, c, strategy):
    dev = _dev()
    q = (1 << m) - c
    rng = random.Random(bits * 7919 + m + c % 1000)
    f = dev.Field(bits, q, strategy)
    assert f.reduction == "special_form"
    g = dev.Field(bits, q, strategy, reduction="barrett")
    assert g.reduction == "barrett"
    xs, ys = _operands(rng, q, 3000)
    want = [a * b % q for a, b in zip(xs, ys)]
    assert _run(f, "vmul", xs, ys) == want
    assert _run(g, "vmul", xs, ys) == want
    for s in (0, 1, q - 1, rng.randrange(q)):
        want = [(s * a + b) % q for a, b in zip(xs, ys)]
        assert _run(f, "axpy", xs, ys, s) == want
        assert _run(g, "axpy", xs, ys, s) == want


def test_reduction_selection(cuda):
    """Moduli outside the special form keep the Barrett path; full-width
    fields stay Montgomery."""
    dev = _dev()
    from paper_2501_07535_b200.params import find_ntt_params
    for bits in (128, 256, 384, 768):
        assert dev.Field(bits, find_ntt_params(bits, 1).p).reduction == "special_form"
        assert dev.Field(bits, find_ntt_params(bits, 1 << 16).p).reduction == "special_form"
    rng = random.Random(5)
    q = rng.randrange(1 << 250, 1 << 251) | 1  # c = 2^251 - q spans many limbs
    assert dev.Field(256, q).reduction == "barrett"
    assert dev.Field(64, find_ntt_params(64, 1).p).reduction == "barrett"  # m = 60 < 72
    assert dev.Field(256, (1 << 255) - 19, "montgomery").reduction == "montgomery"
    with pytest.raises(ValueError):
        dev.Field(256, (1 << 255) - 19, "montgomery", reduction="barrett")
    with pytest.raises(ValueError):
        dev.Field(256, 1 << 200 | 1, reduction="fast")


@pytest.mark.parametrize("bits,logn,batch", [(128, 10, 3), (256, 12, 2), (256, 16, 1), (384, 11, 2),
                                             (768, 10, 2), (1024, 9, 1), (256, 18, 1)])
def test_ntt_special_form_equals_barrett_and_oracle(cuda, bits, logn, batch):
    """The same transform with two-fold butterflies (MODE 3) and Shoup
    butterflies (MODE 0, reduction="barrett") equals the C oracle's run_ntt."""
    dev = _dev()
    from paper_2501_07535_b200.params import find_ntt_params
    n = 1 << logn
    prm = find_ntt_params(bits, n)
    fa = dev.Field(bits, prm.p)
    fb = dev.Field(bits, prm.p, reduction="barrett")
    assert fa.reduction == "special_form" and fb.reduction == "barrett"
    pa, pb = dev.NttPlan(fa, prm), dev.NttPlan(fb, prm)
    rng = np.random.Generator(np.random.PCG64(logn * 31 + bits))
    xs = bigint.uniform_residues(rng, batch * n, prm.p)
    xl = dev.ints_to_limbs(xs, fa.limbs)
    x = dev.to_device(xl)
    ya, yb = pa.forward(x), pb.forward(x)
    assert np.array_equal(dev.to_host(ya), dev.to_host(yb))
    if n <= 1 << 16:
        of = OracleField(prm.p, bits)
        assert np.array_equal(dev.to_host(ya), of.ntt(xl, n, prm.root))
    za, zb = pa.inverse(ya), pb.inverse(yb)
    assert np.array_equal(dev.to_host(za), xl)
    assert np.array_equal(dev.to_host(zb), xl)


def test_ntt_special_form_extreme_c(cuda):
    """An NTT over a special-form prime with a large c (p = 2^m - c, c close
    to 2^32): the fold bounds are tightest there."""
    dev = _dev()
    from paper_2501_07535_b200.params import NttParams
    n = 1 << 10
    # largest prime p = 1 mod n below 2^124 with c = 2^124 - p >= 2^31
    m = 124
    k = ((1 << m) - (1 << 31)) // n
    while True:
        p = k * n + 1
        if bigint.is_prime(p):
            break
        k -= 1
    assert (1 << 31) <= (1 << m) - p < (1 << 32)
    g = 2
    while True:
        w = pow(g, (p - 1) // n, p)
        if pow(w, n // 2, p) != 1:
            break
        g += 1
    prm = NttParams(n=n, p=p, root=w, root_inv=pow(w, -1, p), n_inv=pow(n, -1, p))
    f = dev.Field(128, p)
    assert f.reduction == "special_form"
    plan = dev.NttPlan(f, prm)
    rng = np.random.Generator(np.random.PCG64(99))
    xs = bigint.uniform_residues(rng, 4 * n, p)
    xs[:n] = [p - 1] * n  # all-maximal line
    xl = dev.ints_to_limbs(xs, f.limbs)
    y = plan.forward(dev.to_device(xl))
    of = OracleField(p, 128)
    assert np.array_equal(dev.to_host(y), of.ntt(xl, n, w))
    assert np.array_equal(dev.to_host(plan.inverse(y)), xl)


def test_convolve_special_form_equals_barrett(cuda):
    dev = _dev()
    from paper_2501_07535_b200.params import find_ntt_params
    n = 1 << 14
    prm = find_ntt_params(256, n)
    rng = np.random.Generator(np.random.PCG64(3))
    a = dev.to_device(dev.ints_to_limbs(bigint.uniform_residues(rng, 2 * n, prm.p), 8))
    b = dev.to_device(dev.ints_to_limbs(bigint.uniform_residues(rng, 2 * n, prm.p), 8))
    outs = []
    for red in ("auto", "barrett"):
        plan = dev.NttPlan(dev.Field(256, prm.p, reduction=red), prm)
        outs.append(dev.to_host(plan.convolve(a, b)))
    assert np.array_equal(outs[0], outs[1])
