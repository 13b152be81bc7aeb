"""Modulus, Barrett and transform-parameter setup (host side).

Mirrors the parameter half of the reference's ``widemod.oracle``
(pkg/src/widemod/oracle.py): the same exception types (17-30), the same
``BarrettParams``/``NttParams`` records (57-82), ``compute_barrett``
(109-134) and ``find_ntt_params`` (186-239) with the same choices — largest
prime p = 1 (mod n) below 2^(width-4) and the *smallest* element of exact
order n as the root — so a kernel built here sees exactly the modulus and root
the reference would bake in.  The device kernels then use their own reduction
constants (see csrc/wm_limb.cuh); the reference's ``mu``/shifts are kept here
for API parity and for the reference-layout tools.
"""

from __future__ import annotations

import functools
import random
from dataclasses import dataclass


class ZeroModulus(ValueError):
    """Modulus was zero (or negative)."""


class ModulusOutOfRange(ValueError):
    """Modulus violates the reduction-parameter bounds for the width."""


class NoSuitablePrime(ValueError):
    """No prime with the requested residue properties in the scan range."""


class LengthMismatch(ValueError):
    """Sequence operands have different lengths."""


@dataclass(frozen=True)
class BarrettParams:
    """Reduction constants for a modulus just under ``2**mbits``
    (reference oracle.py:57-71)."""

    q: int
    width: int
    mbits: int
    mu: int
    shift1: int
    shift2: int


@dataclass(frozen=True)
class NttParams:
    """Prime and root of unity for length-``n`` transforms (oracle.py:74-82)."""

    n: int
    p: int
    root: int
    root_inv: int
    n_inv: int


def compute_barrett(q: int, width: int) -> BarrettParams:
    """Barrett constants at ``width`` (reference oracle.py:109-134):
    ``mbits = width - 4``, ``2**(mbits-1) < q < 2**mbits``,
    ``mu = floor(2**(2*mbits+3) / q)``, shifts ``mbits-2`` and ``mbits+5``."""
    if q <= 0:
        raise ZeroModulus(f"modulus must be positive, got {q}")
    if width < 8:
        raise ValueError(f"width must be at least 8, got {width}")
    mbits = width - 4
    lo, hi = 1 << (mbits - 1), 1 << mbits
    if not lo < q < hi:
        raise ModulusOutOfRange(
            f"need 2**{mbits - 1} < q < 2**{mbits} for width {width}, got q={q}")
    mu = (1 << (2 * mbits + 3)) // q
    if mu.bit_length() > width:
        raise ModulusOutOfRange(f"mu={mu} does not fit in {width} bits")
    return BarrettParams(q=q, width=width, mbits=mbits, mu=mu,
                         shift1=mbits - 2, shift2=mbits + 5)


# Trial-division primes; also the deterministic Miller-Rabin bases, which are
# exact for every n < 3.3e24 (and so for every n < 2**64).
_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def _mr_round(n: int, d: int, s: int, a: int) -> bool:
    """One strong-probable-prime round; True when n passes base a."""
    x = pow(a, d, n)
    if x == 1 or x == n - 1:
        return True
    for _ in range(s - 1):
        x = x * x % n
        if x == n - 1:
            return True
    return False


def is_prime(n: int) -> bool:
    """Miller-Rabin with the reference's witness schedule (oracle.py:152-183):
    fixed bases below 2**64, otherwise 40 bases drawn from ``Random(n)``."""
    if n < 2:
        return False
    for b in _BASES:
        if n % b == 0:
            return n == b
    d, s = n - 1, 0
    while not d & 1:
        d >>= 1
        s += 1
    if n < 1 << 64:
        bases = [b for b in _BASES if b < n - 1]
    else:
        rng = random.Random(n)
        bases = [rng.randrange(2, n - 1) for _ in range(40)]
    return all(_mr_round(n, d, s, b) for b in bases)


def _order_n_seed(p: int, n: int) -> int:
    """First g^((p-1)/n), g = 2, 3, ..., whose order is exactly n."""
    e = (p - 1) // n
    half = n // 2
    for g in range(2, p):
        c = pow(g, e, p)
        if c != 1 and pow(c, half, p) != 1:
            return c
    raise NoSuitablePrime(f"no element of order {n} mod {p}")


def _smallest_exact_order(seed: int, p: int, n: int) -> int:
    """min over the odd powers seed^(2i+1), i < n/2 — exactly the elements of
    order n (reference oracle.py:229-237)."""
    step = seed * seed % p
    best = x = seed
    for _ in range(n // 2 - 1):
        x = x * step % p
        if x < best:
            best = x
    return best


@functools.lru_cache(maxsize=64)
def find_ntt_params(width: int, n: int) -> NttParams:
    """Largest prime p = 1 (mod n) with 2**(width-5) < p < 2**(width-4) and
    the smallest root of exact order n (reference oracle.py:186-239)."""
    if width < 8:
        raise ValueError(f"width must be at least 8, got {width}")
    if n < 1 or n & (n - 1):
        raise ValueError(f"transform length must be a power of two, got {n}")
    top = (1 << (width - 4)) - 1
    floor_ = (1 << (width - 5)) + 1
    p = top - (top - 1) % n
    while p >= floor_ and not is_prime(p):
        p -= n
    if p < floor_:
        raise NoSuitablePrime(
            f"no prime p = 1 (mod {n}) with 2**{width - 5} < p < 2**{width - 4}")
    root = 1 if n == 1 else _smallest_exact_order(_order_n_seed(p, n), p, n)
    return NttParams(n=n, p=p, root=root, root_inv=pow(root, -1, p),
                     n_inv=pow(n, -1, p))
