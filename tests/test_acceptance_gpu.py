"""Device analogues of the reference acceptance criteria for the hot path
(reference tests/test_acceptance.py): C1 exhaustive Barrett
at width 8, C2 16-bit add/sub/mul on edges + 100k random pairs, C3 64-bit
mulmod on 10k random pairs, C5 NTT roundtrip / convolution / delta over the
reference's NTT_CONFIGS x 100 vectors.  Same seeds as the reference (1337)."""

from __future__ import annotations

import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED = 1337  # test_acceptance.py:35
NTT_CONFIGS = [(16, 8, 4), (16, 8, 8), (16, 8, 16), (16, 8, 32), (16, 8, 64),
               (128, 64, 4), (128, 64, 16)]  # test_acceptance.py:36-37


def _ops(bits, q, xs, ys):
    from paper_2501_07535_b200 import device as dev
    f = dev.Field(bits, q)
    x = dev.to_device(dev.ints_to_limbs(xs, f.limbs))
    y = dev.to_device(dev.ints_to_limbs(ys, f.limbs))
    return {k: dev.limbs_to_ints(dev.to_host(getattr(f, k)(x, y))) for k in ("vadd", "vsub", "vmul")}


def test_c1_exhaustive_width8(cuda):  # test_acceptance.py:132-152
    total = 0
    for q in range(9, 16):
        xs = [a for a in range(q) for _ in range(q)]
        ys = [b for _ in range(q) for b in range(q)]
        got = _ops(8, q, xs, ys)
        assert got["vmul"] == [a * b % q for a, b in zip(xs, ys)]
        assert got["vadd"] == [(a + b) % q for a, b in zip(xs, ys)]
        assert got["vsub"] == [(a - b) % q for a, b in zip(xs, ys)]
        total += q * q
    assert total == 1036  # sum_{q=9..15} q^2, the reference's C1 case count


def test_c2_16bit_edges_and_100k(cuda):  # test_acceptance.py:155-175
    rnd = random.Random(SEED)
    q = 4093
    edges = [(a, b) for a in (0, 1, q - 1) for b in (0, 1, q - 1)]
    for kind, ref in (("vadd", lambda a, b: (a + b) % q), ("vsub", lambda a, b: (a - b) % q),
                      ("vmul", lambda a, b: a * b % q)):
        cases = edges + [(rnd.randrange(q), rnd.randrange(q)) for _ in range(100_000)]
        xs, ys = [a for a, _ in cases], [b for _, b in cases]
        assert _ops(16, q, xs, ys)[kind] == [ref(a, b) for a, b in cases], kind


def test_c3_64bit_mulmod_10k(cuda):  # test_acceptance.py:178-190
    from paper_2501_07535_b200.params import find_ntt_params
    q = find_ntt_params(64, 1).p
    rnd = random.Random(SEED + 1)
    cases = [(rnd.randrange(q), rnd.randrange(q)) for _ in range(10_000)]
    xs, ys = [a for a, _ in cases], [b for _, b in cases]
    assert _ops(64, q, xs, ys)["vmul"] == [a * b % q for a, b in cases]


@pytest.mark.parametrize("bits,word,n", NTT_CONFIGS)
def test_c5_ntt_roundtrip_convolution_delta(cuda, bits, word, n):  # test_acceptance.py:223-250
    from oracle import bigint
    from paper_2501_07535_b200 import device as dev
    from paper_2501_07535_b200 import kernels as K
    fwd = K.generate_kernel(K.make_spec("ntt", bits, word, size=n))
    plan = fwd.plan()
    p = plan.params.p
    rnd = random.Random(SEED + bits + n)
    vecs = [[rnd.randrange(p) for _ in range(n)] for _ in range(100)]
    X = dev.to_device(dev.ints_to_limbs([v for vec in vecs for v in vec], plan.limbs))
    Y = plan.forward(X)
    back = plan.inverse(Y)
    assert np.array_equal(dev.to_host(back), dev.to_host(X)), "roundtrip"
    # convolution of consecutive pairs, fused device path vs direct summation
    A = X[: 2 * n].contiguous()
    B = X[2 * n: 4 * n].contiguous()
    conv = dev.limbs_to_ints(dev.to_host(plan.convolve(A, B)))
    for t in range(2):
        assert conv[t * n:(t + 1) * n] == bigint.convolve_mod(vecs[t], vecs[2 + t], p)
    # delta -> all ones; ones -> (n, 0, ..., 0)
    assert K.run_ntt(fwd, [1] + [0] * (n - 1)) == [1] * n
    assert K.run_ntt(fwd, [1] * n) == [n % p] + [0] * (n - 1)


def test_convolve_large_and_aliasing(cuda):
    """Fused convolution at 256-bit n=2^16 (2 passes) and n=2^12, against the
    unfused NTT -> vmul -> INTT sequence; a may alias out."""
    import torch
    from paper_2501_07535_b200 import kernels as K
    from paper_2501_07535_b200.params import find_ntt_params
    for logn, batch in ((12, 3), (16, 2)):
        n = 1 << logn
        plan = K.get_plan(256, find_ntt_params(256, n))
        g = torch.Generator(device="cuda").manual_seed(logn)
        a = torch.randint(-(1 << 31), 1 << 31, (batch * n, 8), dtype=torch.int32, device="cuda", generator=g)
        b = torch.randint(-(1 << 31), 1 << 31, (batch * n, 8), dtype=torch.int32, device="cuda", generator=g)
        a[:, 7] &= (1 << 27) - 1
        b[:, 7] &= (1 << 27) - 1
        want = plan.inverse(plan.field.vmul(plan.forward(a), plan.forward(b)))
        assert torch.equal(plan.convolve(a, b), want)
        a2 = a.clone()
        plan.convolve(a2, b, out=a2)
        assert torch.equal(a2, want)
        with pytest.raises(ValueError):
            plan.convolve(a, b, out=b)
