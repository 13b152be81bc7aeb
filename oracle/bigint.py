"""TEST INFRASTRUCTURE ONLY — pure-Python restatement of the reference's
big-integer semantics for the hot path.  Each function cites the reference
lines it restates (paths relative to /root/reference/pkg/src/widemod/).
Used as the checker; never imported by the product package.
"""

from __future__ import annotations

import random

import numpy as np


# ------------------------------------------------------------ oracle.py
def modop(kind: str, a: int, b: int, q: int) -> int:
    """oracle.py:85-106 — canonical (a op b) mod q."""
    if q <= 1:
        raise ValueError("modulus must exceed 1")
    if kind == "add":
        return (a + b) % q
    if kind == "sub":
        return (a - b) % q
    if kind == "mul":
        return a * b % q
    if kind == "pow":
        return pow(a, b, q)
    raise ValueError(kind)


def compute_barrett(q: int, width: int) -> tuple[int, int, int, int]:
    """oracle.py:109-134 — returns (mbits, mu, shift1, shift2)."""
    mbits = width - 4
    assert (1 << (mbits - 1)) < q < (1 << mbits), "modulus out of Barrett range"
    return mbits, (1 << (2 * mbits + 3)) // q, mbits - 2, mbits + 5


def barrett_mulmod(a: int, b: int, q: int, width: int) -> int:
    """oracle.py:137-149 / kernels._emit_mulmod kernels.py:140-153."""
    _, mu, s1, s2 = compute_barrett(q, width)
    t = a * b
    r = ((t >> s1) * mu) >> s2
    t -= r * q
    return t - q if t >= q else t


def is_prime(n: int) -> bool:
    """oracle.py:152-183 (same witness schedule)."""
    small = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)
    if n < 2:
        return False
    for p in small:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    if n < 1 << 64:
        wit = [a for a in small if a < n - 1]
    else:
        rng = random.Random(n)
        wit = [rng.randrange(2, n - 1) for _ in range(40)]
    for a in wit:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def find_ntt_params(width: int, n: int) -> dict:
    """oracle.py:186-239 — largest p = 1 (mod n) in (2^(w-5), 2^(w-4)),
    smallest root of exact order n.  Returns a dict n/p/root/root_inv/n_inv."""
    hi = (1 << (width - 4)) - 1
    lo = (1 << (width - 5)) + 1
    p = hi - (hi - 1) % n
    while p >= lo and not is_prime(p):
        p -= n
    if p < lo:
        raise ValueError("no suitable prime")
    if n == 1:
        root = 1
    else:
        seed = 0
        for base in range(2, p):
            c = pow(base, (p - 1) // n, p)
            if c != 1 and pow(c, n // 2, p) != 1:
                seed = c
                break
        sq = seed * seed % p
        root = x = seed
        for _ in range(n // 2 - 1):
            x = x * sq % p
            root = min(root, x)
    return {"n": n, "p": p, "root": root, "root_inv": pow(root, -1, p), "n_inv": pow(n, -1, p)}


def convolve_mod(f: list[int], g: list[int], p: int) -> list[int]:
    """oracle.py:242-259 — direct cyclic convolution."""
    n = len(f)
    assert len(g) == n
    return [sum(f[i] * g[(k - i) % n] for i in range(n)) % p for k in range(n)]


def ntt_reference(vec: list[int], p: int, root: int, root_inv: int, n_inv: int,
                  inverse: bool = False) -> list[int]:
    """oracle.py:262-282 — direct O(n^2) DFT."""
    n = len(vec)
    w = root_inv if inverse else root
    out = []
    for k in range(n):
        acc = sum(x * pow(w, j * k, p) for j, x in enumerate(vec)) % p
        out.append(acc * n_inv % p if inverse else acc)
    return out


# ------------------------------------------------------------ kernels.py executors
def addmod(a: int, b: int, q: int) -> int:
    """kernels._emit_addmod kernels.py:122-128: s<q ? s : s-q."""
    s = a + b
    return s if s < q else s - q


def submod(a: int, b: int, q: int) -> int:
    """kernels._emit_submod kernels.py:131-137: a<b ? a-b+q : a-b."""
    return a - b + q if a < b else a - b


def run_vector(kind: str, q: int, width: int, *arrays) -> list[int]:
    """kernels.run_vector kernels.py:467-480 over build_vector kernels.py:215-256."""
    if kind == "vadd":
        return [addmod(a, b, q) for a, b in zip(*arrays)]
    if kind == "vsub":
        return [submod(a, b, q) for a, b in zip(*arrays)]
    if kind == "vmul":
        return [barrett_mulmod(a, b, q, width) for a, b in zip(*arrays)]
    if kind == "axpy":
        s, xs, ys = arrays
        return [addmod(barrett_mulmod(s, x, q, width), y, q) for x, y in zip(xs, ys)]
    raise ValueError(kind)


def twiddle_table(p: int, n: int, base: int) -> list[int]:
    """kernels.twiddle_table kernels.py:259-267."""
    out, acc = [], 1
    for _ in range(max(1, n // 2)):
        out.append(acc)
        acc = acc * base % p
    return out


def bit_reverse_order(n: int) -> list[int]:
    """kernels.bit_reverse_order kernels.py:386-392."""
    bits = (n - 1).bit_length()
    if n == 1:
        return [0]
    return [int(format(i, f"0{bits}b")[::-1], 2) for i in range(n)]


def run_ntt(values: list[int], prm: dict, width: int, inverse: bool = False) -> list[int]:
    """kernels.run_ntt kernels.py:483-499 with butterfly_schedule kernels.py:395-413
    and the build_ntt butterfly kernels.py:290-292 (u + v*w, u - v*w)."""
    n, p = prm["n"], prm["p"]
    tw = twiddle_table(p, n, prm["root_inv"] if inverse else prm["root"])
    rev = bit_reverse_order(n)
    x = [values[rev[i]] for i in range(n)]
    m = 2
    while m <= n:
        half, step = m // 2, n // m
        for base in range(0, n, m):
            for j in range(half):
                u, v = x[base + j], x[base + j + half]
                t = barrett_mulmod(v, tw[j * step], p, width)
                x[base + j] = addmod(u, t, p)
                x[base + j + half] = submod(u, t, p)
        m *= 2
    if inverse:
        x = [addmod(0, barrett_mulmod(v, prm["n_inv"], p, width), p) for v in x]
    return x


def run_ntt_exact(values: list[int], p: int, root: int, n_inv: int, inverse: bool = False) -> list[int]:
    """run_ntt (kernels.py:483-499) with exact modular products instead of the
    reference's width-bound Barrett: the same bit-reversal, butterfly schedule
    and inverse scaling, valid for any prime p (full-width moduli, which the
    reference's compute_barrett range excludes).  `root` is root_inv for the
    inverse; agrees with run_ntt wherever both apply (tests/test_oracle_pinned.py)."""
    n = len(values)
    tw = [pow(root, e, p) for e in range(n // 2)]
    rev = bit_reverse_order(n)
    x = [values[rev[i]] for i in range(n)]
    m = 2
    while m <= n:
        half, step = m // 2, n // m
        for base in range(0, n, m):
            for j in range(half):
                u, v = x[base + j], x[base + j + half]
                t = v * tw[j * step] % p
                x[base + j] = (u + t) % p
                x[base + j + half] = (u - t) % p
        m *= 2
    if inverse:
        x = [v * n_inv % p for v in x]
    return x


def ntt_point(values: list[int], p: int, root: int, k: int) -> int:
    """y[k] = sum_j x[j] root^(jk) mod p by Horner (the DFT ntt_reference,
    oracle.py:262-282, at one output index)."""
    w = pow(root, k, p)
    acc = 0
    for x in reversed(values):
        acc = (acc * w + x) % p
    return acc


# ------------------------------------------------------------ inputs
def uniform_residues(rng: np.random.Generator, count: int, q: int) -> list[int]:
    """Uniform values in [0, q): k uint32 limbs per value, top limb masked to
    the modulus bit length, rejection of values >= q."""
    k = (q.bit_length() + 31) // 32
    top_bits = q.bit_length() - 32 * (k - 1)
    out: list[int] = []
    while len(out) < count:
        need = count - len(out)
        limbs = rng.integers(0, 1 << 32, size=(need, k), dtype=np.uint64).astype("<u4")
        limbs[:, -1] &= np.uint32((1 << top_bits) - 1)
        raw = limbs.tobytes()
        step = 4 * k
        for i in range(need):
            v = int.from_bytes(raw[i * step:(i + 1) * step], "little")
            if v < q:
                out.append(v)
    return out


def uniform_residue_limbs(rng: np.random.Generator, count: int, q: int, limbs: int | None = None) -> np.ndarray:
    """uniform_residues as a uint32 limb array [count, limbs] (little-endian
    limbs), vectorised: the same draws, the same rejections, the same order
    (pinned equal in tests/test_oracle_pinned.py).  For the full-size parity
    fixtures (2^16 x 64 .. 2^24 elements) where Python ints are too slow."""
    k = (q.bit_length() + 31) // 32
    top_bits = q.bit_length() - 32 * (k - 1)
    qw = [(q >> (32 * j)) & 0xFFFFFFFF for j in range(k)]
    parts = []
    have = 0
    while have < count:
        need = count - have
        l = rng.integers(0, 1 << 32, size=(need, k), dtype=np.uint64).astype("<u4")
        l[:, -1] &= np.uint32((1 << top_bits) - 1)
        gt = np.zeros(need, dtype=bool)
        eq = np.ones(need, dtype=bool)
        for j in range(k - 1, -1, -1):
            gt |= eq & (l[:, j] > qw[j])
            eq &= l[:, j] == qw[j]
        keep = l[~(gt | eq)]
        parts.append(keep)
        have += keep.shape[0]
    out = np.concatenate(parts)[:count]
    if limbs is not None and limbs > k:
        out = np.concatenate([out, np.zeros((count, limbs - k), dtype="<u4")], axis=1)
    return np.ascontiguousarray(out)
