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
    # moduli that leave the top limb empty (vmul takes the two-Montgomery-product path)
    (256, M127), (1024, SECP256K1_P), (64, 2**32 - 5),
    # limb counts without Montgomery kernels of their own (zero-padded to 4 / 8 / 16 limbs)
    (96, 2**96 - 17), (160, 2**160 - 47), (480, 2**480 - 65),
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


# ------------------------------------------------------------------ NTT
BN254_R = 21888242871839275222246405745257275088548364400416034343698204186575808495617


def _ntt_prime(bits: int, two_adicity: int, seed: int) -> int:
    """A prime p = c 2^a + 1 with exactly `bits` bits (full width)."""
    from oracle import bigint
    rnd = random.Random(seed)
    while True:
        c = rnd.randrange(2 ** (bits - two_adicity - 1), 2 ** (bits - two_adicity))
        p = c * 2**two_adicity + 1
        if p.bit_length() == bits and bigint.is_prime(p):
            return p


def _params(p: int, n: int):
    from paper_2501_07535_b200.params import NttParams
    assert (p - 1) % n == 0
    x = 2
    while True:  # root of exact order n: x^((p-1)/n) with x a non-residue
        if pow(x, (p - 1) // 2, p) == p - 1:
            break
        x += 1
    root = pow(x, (p - 1) // n, p)
    assert pow(root, n // 2, p) == p - 1
    return NttParams(n=n, p=p, root=root, root_inv=pow(root, -1, p), n_inv=pow(n, -1, p))


_NAMED = {"bls12_381_r": BLS12_381_R, "bn254_r": BN254_R, "goldilocks": GOLDILOCKS}
_PRIMES: dict = {}


def _prime(name: str, bits: int) -> int:
    """Named curve/FHE primes, or a random 2^24-NTT prime of full width
    ("random") or two bits below it ("random2": the NTT's Shoup / [0, 4p)
    mode for full-width fields) (cached)."""
    if name in _NAMED:
        return _NAMED[name]
    if (name, bits) not in _PRIMES:
        _PRIMES[(name, bits)] = _ntt_prime(bits - (2 if name == "random2" else 0), 24, bits)
    return _PRIMES[(name, bits)]


FIELDS = [(256, "bls12_381_r"), (256, "bn254_r"), (64, "goldilocks")] + [
    (bits, "random") for bits in (32, 128, 384, 512, 768, 1024)] + [
    (bits, "random2") for bits in (64, 128, 384, 768, 1024)] + [
    (96, "random"), (160, "random"), (224, "random2")]  # limb counts padded to a Montgomery build


@pytest.mark.parametrize("bits,name", FIELDS)
@pytest.mark.parametrize("logn", [1, 3, 6, 9, 12])
def test_ntt_full_width_vs_exact_oracle(cuda, bits, name, logn):
    from oracle import bigint
    dev = _dev()
    p = _prime(name, bits)
    if bits >= 768 and logn > 9:
        pytest.skip("O(n log n) Python oracle budget")
    n = 1 << logn
    f = dev.Field(bits, p, "montgomery")
    plan = dev.NttPlan(f, _params(p, n))
    prm = plan.params
    rnd = random.Random(bits * 100 + logn)
    batch = 2
    xs = [rnd.randrange(p) for _ in range(batch * n)]
    xs[:3] = [0, 1, p - 1]
    xd = dev.to_device(dev.ints_to_limbs(xs, f.limbs))
    got = dev.limbs_to_ints(dev.to_host(plan.forward(xd)))
    got_i = dev.limbs_to_ints(dev.to_host(plan.inverse(xd)))
    for b in range(batch):
        seg = xs[b * n:(b + 1) * n]
        assert got[b * n:(b + 1) * n] == bigint.run_ntt_exact(seg, p, prm.root, prm.n_inv), (bits, n, b)
        assert got_i[b * n:(b + 1) * n] == bigint.run_ntt_exact(seg, p, prm.root_inv, prm.n_inv, inverse=True)


@pytest.mark.parametrize("bits,name,logn", [(256, "bls12_381_r", 16), (256, "bls12_381_r", 21),
                                             (64, "goldilocks", 22), (1024, "random", 19),
                                             (256, "bn254_r", 21), (768, "random2", 20)])
def test_ntt_full_width_large(cuda, bits, name, logn):
    """Multi-pass plans: INTT(NTT(x)) == x and Horner evaluations of outputs."""
    import torch
    from oracle import bigint
    dev = _dev()
    p = _prime(name, bits)
    n = 1 << logn
    f = dev.Field(bits, p, "montgomery")
    plan = dev.NttPlan(f, _params(p, n))
    rnd = random.Random(logn)
    g = torch.Generator(device="cuda").manual_seed(logn)
    Kl = f.limbs
    x = torch.randint(-(1 << 31), 1 << 31, (n, Kl), dtype=torch.int32, device="cuda", generator=g)
    x[:, Kl - 1] &= (1 << (p.bit_length() - 1 - 32 * (Kl - 1))) - 1  # < 2^(bitlen-1) <= p
    y = plan.forward(x)
    assert torch.equal(plan.inverse(y), x)
    xs = dev.limbs_to_ints(dev.to_host(x))
    yh = dev.to_host(y)
    for k in [0, 1, n - 1, rnd.randrange(n)]:
        assert dev.limbs_to_ints(yh[k:k + 1])[0] == bigint.ntt_point(xs, p, plan.params.root, k), k


def test_full_width_convolution_and_host_pipeline(cuda):
    """NTT-domain convolution (fused pointwise product) and the host-buffer
    pipeline on a full-width field."""
    import torch
    from oracle import bigint
    from paper_2501_07535_b200 import kernels as Kmod
    dev = _dev()
    p, n = BLS12_381_R, 256
    f = dev.Field(256, p, "montgomery")
    plan = dev.NttPlan(f, _params(p, n))
    rnd = random.Random(7)
    a = [rnd.randrange(p) for _ in range(n)]
    b = [rnd.randrange(p) for _ in range(n)]
    got = dev.limbs_to_ints(dev.to_host(plan.convolve(dev.to_device(dev.ints_to_limbs(a, 8)),
                                                      dev.to_device(dev.ints_to_limbs(b, 8)))))
    assert got == bigint.convolve_mod(a, b, p)
    batch = 3
    xs = [rnd.randrange(p) for _ in range(batch * n)]
    import numpy as np
    words_in = [w for v in xs for w in Kmod.to_words(v, 4, 64)]
    host_in = torch.from_numpy(np.array(words_in, dtype=np.uint64).view(np.int64)).pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    plan.host_transform(host_in, host_out, mode="forward", word_bits=64, ref_words=4, chunk=1)
    torch.cuda.synchronize()
    words = host_out.numpy().view("uint64").tolist()
    out = [Kmod.from_words(words[i * 4:(i + 1) * 4], 64) for i in range(batch * n)]
    for t in range(batch):
        seg = xs[t * n:(t + 1) * n]
        assert out[t * n:(t + 1) * n] == bigint.run_ntt_exact(seg, p, plan.params.root, plan.params.n_inv)
    tw = dev.limbs_to_ints(dev.to_host(plan.twiddles(16)))
    assert tw == [pow(plan.params.root, e, p) for e in range(16)]
