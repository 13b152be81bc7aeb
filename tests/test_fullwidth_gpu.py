"""Full-width moduli (WM_FIELD_MONTGOMERY; the paper's Montgomery mode for
moduli of full bit width): vadd/vsub/vmul/axpy bit-exact
against Python big integers for curve / FHE primes that the reference's
Barrett range (q < 2^(bits-4), oracle.py:124-128) excludes, random odd
full-width moduli, and the extreme modulus 2^(32K) - 1."""

from __future__ import annotations

import random

import pytest

pytestmark = pytest.mark.gpu

SECP256K1_P = 2**256 - 2**32 - 977
BLS12_381_R = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001
BN254_P = 21888242871839275222246405745257275088696311157297823662689037894645226208583
BLS12_381_P = int("1a0111ea397fe69a4b1ba7b6434bacd764774b84f38512bf6730d2a0f6b0f6241eabfffeb153ffffb9feffffffffaaab", 16)
GOLDILOCKS = 2**64 - 2**32 + 1
M127 = 2**127 - 1

CASES = [
    (256, SECP256K1_P), (256, BLS12_381_R), (256, BN254_P), (384, BLS12_381_P),
    (64, GOLDILOCKS), (128, M127), (32, 2**32 - 5), (1024, 2**1024 - 1),
    (768, 2**768 - 1), (512, 2**512 - 569),
]


def _dev():
    from paper_2501_07535_b200 import device
    return device


def _run(kind, bits, q, xs, ys, scalar=0):
    dev = _dev()
    f = dev.Field(bits, q, "montgomery")
    x = dev.to_device(dev.ints_to_limbs(xs, f.limbs))
    y = dev.to_device(dev.ints_to_limbs(ys, f.limbs))
    out = f.axpy(scalar, x, y) if kind == "axpy" else getattr(f, kind)(x, y)
    return dev.limbs_to_ints(dev.to_host(out))


def _inputs(q, n, seed):
    rnd = random.Random(seed)
    edges = [0, 1, 2, q - 1, q - 2, q // 2, (q + 1) // 2]
    xs = [rnd.randrange(q) for _ in range(n)] + [a for a in edges for _ in edges]
    ys = [rnd.randrange(q) for _ in range(n)] + [b for _ in edges for b in edges]
    return xs, ys


@pytest.mark.parametrize("bits,q", CASES)
def test_blas_full_width(cuda, bits, q):
    xs, ys = _inputs(q, 3000, bits)
    assert _run("vadd", bits, q, xs, ys) == [(a + b) % q for a, b in zip(xs, ys)]
    assert _run("vsub", bits, q, xs, ys) == [(a - b) % q for a, b in zip(xs, ys)]
    assert _run("vmul", bits, q, xs, ys) == [(a * b) % q for a, b in zip(xs, ys)]
    for s in (0, 1, q - 1, random.Random(q).randrange(q)):
        assert _run("axpy", bits, q, xs, ys, s) == [(s * a + b) % q for a, b in zip(xs, ys)]


@pytest.mark.parametrize("limbs", [1, 2, 4, 8, 12, 16, 24, 32])
def test_random_full_width_moduli(cuda, limbs):
    rnd = random.Random(limbs)
    for _ in range(3):
        bits = 32 * limbs
        q = rnd.randrange(2 ** (bits - 1), 2**bits) | 1  # top bit set, odd
        xs, ys = _inputs(q, 500, q)
        assert _run("vmul", bits, q, xs, ys) == [(a * b) % q for a, b in zip(xs, ys)]
        assert _run("vadd", bits, q, xs, ys) == [(a + b) % q for a, b in zip(xs, ys)]


def test_full_width_field_rejections(cuda):
    dev = _dev()
    with pytest.raises(ValueError):
        dev.Field(256, SECP256K1_P + 1, "montgomery")  # even modulus
    with pytest.raises(ValueError):
        dev.Field(255, SECP256K1_P, "montgomery")  # wider than the stated width
    with pytest.raises(ValueError):
        dev.Field(256, SECP256K1_P)  # Barrett fields keep the reference range
