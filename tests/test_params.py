"""The product's host-side parameter setup (paper_2501_07535_b200.params)
reproduces the reference's moduli, roots and Barrett constants exactly
(golden params.json from the reference's find_ntt_params/compute_barrett, and
the pins of reference tests/test_oracle.py)."""

from __future__ import annotations

import pytest

from paper_2501_07535_b200 import params as P


def test_barrett_pins():  # reference test_oracle.py:54-75
    assert P.compute_barrett(13, 8) == P.BarrettParams(q=13, width=8, mbits=4, mu=157, shift1=2, shift2=9)
    b = P.compute_barrett(4093, 16)
    assert (b.mbits, b.mu, b.shift1, b.shift2) == (12, 32792, 10, 17)
    with pytest.raises(P.ModulusOutOfRange):
        P.compute_barrett(8, 8)
    with pytest.raises(P.ModulusOutOfRange):
        P.compute_barrett(16, 8)
    with pytest.raises(P.ZeroModulus):
        P.compute_barrett(0, 8)
    with pytest.raises(ValueError):
        P.compute_barrett(13, 4)
    P.compute_barrett(9, 8)
    P.compute_barrett(15, 8)


def test_is_prime_pins():  # reference test_oracle.py:96-112
    for n in range(2, 100):
        assert P.is_prime(n) == all(n % d for d in range(2, n))
    assert not P.is_prime(0) and not P.is_prime(1) and not P.is_prime(91)
    assert not P.is_prime(561) and not P.is_prime(341550071728321)
    assert P.is_prime((1 << 61) - 1) and P.is_prime((1 << 89) - 1)
    assert not P.is_prime(((1 << 89) - 1) * ((1 << 61) - 1))


def test_find_ntt_params_pins():  # reference test_oracle.py:115-137
    assert P.find_ntt_params(8, 4) == P.NttParams(n=4, p=13, root=5, root_inv=8, n_inv=10)
    assert P.find_ntt_params(8, 1) == P.NttParams(n=1, p=13, root=1, root_inv=1, n_inv=1)
    with pytest.raises(P.NoSuitablePrime):
        P.find_ntt_params(8, 8)
    with pytest.raises(ValueError):
        P.find_ntt_params(16, 6)
    assert P.find_ntt_params(64, 1).p == 1152921504606846883


def test_params_golden(golden):
    for row in golden("params"):
        if row["n"] > 1 << 20:
            continue  # 2^24 root scan takes ~5 s in Python; covered by the slow test below
        got = P.find_ntt_params(row["width"], row["n"])
        assert (got.p, got.root, got.root_inv, got.n_inv) == (
            int(row["p"]), int(row["root"]), int(row["root_inv"]), int(row["n_inv"]))
        b = P.compute_barrett(got.p, row["width"])
        assert (b.mu, b.mbits, b.shift1, b.shift2) == (int(row["mu"]), row["mbits"], row["shift1"], row["shift2"])


def test_params_golden_2p24(golden):
    row = [r for r in golden("params") if r["n"] == 1 << 24][0]
    got = P.find_ntt_params(row["width"], row["n"])
    assert (got.p, got.root) == (int(row["p"]), int(row["root"]))


@pytest.mark.parametrize("width,n", [(8, 4), (16, 8), (16, 64), (32, 16), (128, 16), (1024, 4)])
def test_find_ntt_params_invariants(width, n):  # reference test_oracle.py:140-150
    got = P.find_ntt_params(width, n)
    assert (1 << (width - 5)) < got.p < (1 << (width - 4))
    assert got.p % n == 1 or n == 1
    assert pow(got.root, n, got.p) == 1
    if n > 1:
        assert pow(got.root, n // 2, got.p) != 1
    assert got.root * got.root_inv % got.p == 1
    assert n * got.n_inv % got.p == 1


def test_root_is_smallest_of_exact_order():  # reference test_oracle.py:153-157
    got = P.find_ntt_params(8, 4)
    cands = [x for x in range(1, 13) if pow(x, 4, 13) == 1 and pow(x, 2, 13) != 1]
    assert got.root == min(cands)
