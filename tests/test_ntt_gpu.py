"""Parity of the sm_100a NTT/INTT with the oracle through the C ABI:
reference golden transforms, the reference's 2^16 256-bit checksums, the C
oracle at 2^20, and size-independent properties (roundtrip, random-point
evaluation, convolution, linearity) at 2^24.  Bit-exact (integer work)."""

from __future__ import annotations

import hashlib
import random

import numpy as np
import pytest

from oracle import bigint
from oracle.cbind import OracleField

pytestmark = pytest.mark.gpu


def _dev():
    from paper_2501_07535_b200 import device
    return device


def plan_for(bits, n):
    from paper_2501_07535_b200 import kernels as K
    from paper_2501_07535_b200.params import find_ntt_params
    return K.get_plan(bits, find_ntt_params(bits, n))


def test_reference_pins(cuda):  # reference test_kernels.py:156-171
    from paper_2501_07535_b200 import kernels as K
    from paper_2501_07535_b200.params import find_ntt_params
    prm = find_ntt_params(8, 4)
    fwd = K.build_program(K.KernelSpec("ntt", K.WordLayout(8, 8), 4, K.compute_barrett(prm.p, 8), prm))
    assert K.run_ntt(fwd, [1, 0, 0, 0]) == [1, 1, 1, 1]
    assert K.run_ntt(fwd, [1, 1, 1, 1]) == [4, 0, 0, 0]
    assert K.run_ntt(fwd, [1, 2, 3, 4]) == [10, 1, 11, 8]
    inv = K.build_program(K.KernelSpec("intt", K.WordLayout(8, 8), 4, K.compute_barrett(prm.p, 8), prm))
    r = random.Random(3)
    for _ in range(25):
        vec = [r.randrange(13) for _ in range(4)]
        assert K.run_ntt(inv, K.run_ntt(fwd, vec)) == vec


def test_golden_transforms(cuda, golden):
    """Reference run_ntt outputs (lowered reference kernels) at 16..768 bits."""
    from paper_2501_07535_b200 import kernels as K
    for row in golden("ntt"):
        fwd = K.generate_kernel(K.make_spec("ntt", row["bits"], row["word"], size=row["n"]))
        inv = K.generate_kernel(K.make_spec("intt", row["bits"], row["word"], size=row["n"]))
        x = [int(v) for v in row["x"]]
        assert K.run_ntt(fwd, x) == [int(v) for v in row["fwd"]], (row["bits"], row["n"])
        assert K.run_ntt(inv, x) == [int(v) for v in row["inv"]], (row["bits"], row["n"])


def test_reference_2p16_checksums(cuda, golden):
    """BASELINE config 2 size: 256-bit n=2^16 forward and inverse equal the
    reference's own run_ntt output (sha256 of the limbs, make_golden.py)."""
    dev = _dev()
    for row in golden("ntt_large"):
        n, p = row["n"], int(row["p"])
        plan = plan_for(256, n)
        x = bigint.uniform_residues(np.random.Generator(np.random.PCG64(row["seed"])), n, p)
        xl = dev.ints_to_limbs(x, 8)
        assert hashlib.sha256(xl.tobytes()).hexdigest() == row["x_sha256"]
        xd = dev.to_device(xl)
        yf = dev.to_host(plan.forward(xd))
        assert hashlib.sha256(yf.tobytes()).hexdigest() == row["fwd_sha256"]
        yi = dev.to_host(plan.inverse(xd))
        assert hashlib.sha256(yi.tobytes()).hexdigest() == row["inv_sha256"]


@pytest.mark.parametrize("bits", [16, 32, 64, 96, 128, 192, 256, 288, 320, 352, 384, 416, 448, 480, 512, 640, 768, 992, 1024])
@pytest.mark.parametrize("logn", [1, 2, 3, 5, 8, 10, 11, 12, 14])
def test_sizes_and_widths_vs_c_oracle(cuda, bits, logn):
    """Every pass structure (1-3 passes) at every built width, batch 3, against
    the C restatement of run_ntt."""
    from paper_2501_07535_b200.params import NoSuitablePrime
    dev = _dev()
    n = 1 << logn
    try:
        plan = plan_for(bits, n)
    except NoSuitablePrime:
        pytest.skip("no prime for this (width, n)")
    prm = plan.params
    of = OracleField(prm.p, bits)
    batch = 3
    rng = np.random.Generator(np.random.PCG64(bits + logn))
    vals = bigint.uniform_residues(rng, batch * n, prm.p)
    kn = (bits + 31) // 32  # oracle limbs; the device may store zero-padded limbs
    xl = dev.ints_to_limbs(vals, kn)
    xd = dev.to_device(dev.ints_to_limbs(vals, plan.limbs))
    for inverse in (False, True):
        got = dev.to_host(plan.inverse(xd) if inverse else plan.forward(xd))
        want = of.ntt(xl, n, prm.root_inv, prm.n_inv) if inverse else of.ntt(xl, n, prm.root)
        assert np.array_equal(got[:, :kn], want), (bits, n, inverse)
        assert not got[:, kn:].any(), (bits, n, "padding limbs")


def test_2p20_vs_c_oracle(cuda):
    """BASELINE config 4 size (256-bit n=2^20), one transform each way."""
    dev = _dev()
    n = 1 << 20
    plan = plan_for(256, n)
    prm = plan.params
    of = OracleField(prm.p, 256)
    xl = dev.ints_to_limbs(bigint.uniform_residues(np.random.Generator(np.random.PCG64(20)), n, prm.p), 8)
    xd = dev.to_device(xl)
    assert np.array_equal(dev.to_host(plan.forward(xd)), of.ntt(xl, n, prm.root))
    assert np.array_equal(dev.to_host(plan.inverse(xd)), of.ntt(xl, n, prm.root_inv, prm.n_inv))


def test_2p24_properties(cuda):
    """BASELINE config 5 size (256-bit n=2^24): random-point evaluation of the
    forward output against the O(n) Horner oracle, and INTT(NTT(x)) == x."""
    dev = _dev()
    import torch
    n = 1 << 24
    plan = plan_for(256, n)
    prm = plan.params
    g = torch.Generator(device="cuda").manual_seed(24)
    x = torch.randint(-(1 << 31), 1 << 31, (n, 8), dtype=torch.int32, device="cuda", generator=g)
    x[:, 7] &= (1 << 27) - 1  # < 2^251 < p: canonical
    y = plan.forward(x)
    back = plan.inverse(y)
    assert torch.equal(back, x)
    of = OracleField(prm.p, 256)
    rnd = random.Random(24)
    ks = [0, 1, n - 1, n // 2] + [rnd.randrange(n) for _ in range(4)]
    pts = of.ntt_points(dev.to_host(x), prm.root, ks)
    yh = dev.to_host(y)
    for i, k in enumerate(ks):
        assert np.array_equal(yh[k], pts[i]), k


@pytest.mark.parametrize("bits,logn", [(512, 21), (768, 21), (1024, 19)])
def test_wide_three_pass_properties(cuda, bits, logn):
    """Three-pass plans at the widest limb counts (radix-2 in-smem stages at
    24 and 32 limbs): INTT(NTT(x)) == x and random-point evaluations of the
    forward output against the O(n) Horner oracle."""
    dev = _dev()
    import torch
    n = 1 << logn
    plan = plan_for(bits, n)
    assert len(plan.pass_log_sizes) == 3, plan.pass_log_sizes
    prm = plan.params
    Kl = plan.limbs
    g = torch.Generator(device="cuda").manual_seed(bits + logn)
    x = torch.randint(-(1 << 31), 1 << 31, (n, Kl), dtype=torch.int32, device="cuda", generator=g)
    x[:, Kl - 1] &= (1 << (bits - 5 - 32 * (Kl - 1))) - 1  # < 2^(bits-5) < p
    y = plan.forward(x)
    assert torch.equal(plan.inverse(y), x)
    of = OracleField(prm.p, bits)
    rnd = random.Random(bits)
    ks = [0, 1, n - 1] + [rnd.randrange(n) for _ in range(3)]
    pts = of.ntt_points(dev.to_host(x), prm.root, ks)
    yh = dev.to_host(y)
    for i, k in enumerate(ks):
        assert np.array_equal(yh[k], pts[i]), k


def test_convolution_and_linearity(cuda):
    """NTT -> pointwise vmul -> INTT equals the cyclic convolution (reference
    verify.py:217-223), and NTT(a x + y) = a NTT(x) + NTT(y)."""
    dev = _dev()
    for bits, n in [(128, 64), (256, 256), (384, 32)]:
        plan = plan_for(bits, n)
        prm = plan.params
        f = plan.field
        rnd = random.Random(bits)
        xs = [rnd.randrange(prm.p) for _ in range(n)]
        ys = [rnd.randrange(prm.p) for _ in range(n)]
        X = plan.forward(dev.to_device(dev.ints_to_limbs(xs, plan.limbs)))
        Y = plan.forward(dev.to_device(dev.ints_to_limbs(ys, plan.limbs)))
        conv = dev.limbs_to_ints(dev.to_host(plan.inverse(f.vmul(X, Y))))
        assert conv == bigint.convolve_mod(xs, ys, prm.p)
        a = rnd.randrange(prm.p)
        lhs = plan.forward(f.axpy(a, dev.to_device(dev.ints_to_limbs(xs, plan.limbs)),
                                  dev.to_device(dev.ints_to_limbs(ys, plan.limbs))))
        rhs = f.axpy(a, X, Y)
        assert np.array_equal(dev.to_host(lhs), dev.to_host(rhs))


def test_device_twiddles_match_twiddle_table(cuda):
    from paper_2501_07535_b200 import kernels as K
    dev = _dev()
    for bits, n in [(16, 8), (256, 1024), (256, 1 << 16), (768, 64)]:
        plan = plan_for(bits, n)
        for inverse in (False, True):
            got = dev.limbs_to_ints(dev.to_host(plan.twiddles(inverse=inverse)))
            assert got == K.twiddle_table(plan.params, inverse=inverse), (bits, n, inverse)


def test_in_place_batch_and_workspace(cuda):
    dev = _dev()
    import torch
    n = 1 << 16
    plan = plan_for(256, n)
    prm = plan.params
    batch = 5
    xl = dev.ints_to_limbs(bigint.uniform_residues(np.random.Generator(np.random.PCG64(9)), batch * n, prm.p), 8)
    ref = dev.to_host(plan.forward(dev.to_device(xl)))
    xd = dev.to_device(xl)
    ws = torch.empty(plan.workspace_bytes(batch) // 4, dtype=torch.int32, device="cuda")
    plan.forward(xd, out=xd, workspace=ws)
    assert np.array_equal(dev.to_host(xd), ref)
    of = OracleField(prm.p, 256)
    assert np.array_equal(ref[n:2 * n], of.ntt(xl[n:2 * n], n, prm.root))
    with pytest.raises(ValueError):
        plan.forward(dev.to_device(xl[: n - 1]))


@pytest.mark.parametrize("mode", ["forward", "inverse", "forward_inverse", "copy"])
def test_host_pipeline_reference_layout(cuda, mode):
    """wm_ntt_host: pinned host buffers in the reference AoS MSW-first layout
    through the chunked H2D / kernels / D2H pipeline equal the device path."""
    dev = _dev()
    import torch
    from paper_2501_07535_b200 import kernels as K
    n, batch = 1 << 12, 7
    plan = plan_for(256, n)
    prm = plan.params
    xs = bigint.uniform_residues(np.random.Generator(np.random.PCG64(31)), batch * n, prm.p)
    ref_words = [w for v in xs for w in K.to_words(v, 4, 64)]
    host_in = torch.from_numpy(np.array(ref_words, dtype=np.uint64).view(np.int64)).pin_memory()
    host_out = torch.empty(host_in.shape, dtype=host_in.dtype, pin_memory=True)
    for chunk in (0, 1, 3, 7):
        host_out.zero_()
        plan.host_transform(host_in, host_out, mode=mode, word_bits=64, ref_words=4, chunk=chunk)
        torch.cuda.synchronize()
        words = host_out.numpy().view(np.uint64).tolist()
        got = [K.from_words(words[i * 4:(i + 1) * 4], 64) for i in range(batch * n)]
        xd = dev.to_device(dev.ints_to_limbs(xs, 8))
        if mode == "forward":
            want = plan.forward(xd)
        elif mode == "inverse":
            want = plan.inverse(xd)
        else:  # forward_inverse round trip, or the copy-only pipeline
            want = xd
        assert got == dev.limbs_to_ints(dev.to_host(want)), chunk


def test_host_pipeline_ramped_chunks(cuda):
    """Auto chunking at n = 2^16 (8 MiB chunks of 4 transforms, halved to 2
    and 1 at both ends): batch 13 -> chunks 1,2,4,3,2,1; in place."""
    dev = _dev()
    import torch
    n, batch = 1 << 16, 13
    plan = plan_for(256, n)
    g = torch.Generator(device="cuda").manual_seed(13)
    x = torch.randint(-(1 << 31), 1 << 31, (batch * n, 8), dtype=torch.int32, device="cuda", generator=g)
    x[:, 7] &= (1 << 27) - 1
    ref = plan.field.to_ref_layout(x, 64, 4).cpu().pin_memory()
    buf = ref.clone().pin_memory()
    plan.host_transform(buf, buf, mode="forward", word_bits=64, ref_words=4)
    torch.cuda.synchronize()
    want = plan.field.to_ref_layout(plan.forward(x), 64, 4).cpu()
    assert torch.equal(buf, want)


def test_host_pipeline_repeated_calls(cuda):
    """Repeated wm_ntt_host calls on the same buffers with new data and
    changing shapes (the slot pool grows and is reused) stay exact."""
    dev = _dev()
    import torch
    n = 1 << 12
    plan = plan_for(256, n)
    f = plan.field
    for batch, chunk in ((9, 0), (9, 0), (9, 2), (9, 0), (5, 0)):
        g = torch.Generator(device="cuda").manual_seed(batch * 10 + chunk)
        x = torch.randint(-(1 << 31), 1 << 31, (batch * n, 8), dtype=torch.int32, device="cuda", generator=g)
        x[:, 7] &= (1 << 27) - 1
        want = f.to_ref_layout(plan.forward(x), 64, 4).cpu()
        for _ in range(3):
            host_in = getattr(test_host_pipeline_repeated_calls, "_hin", None)
            if host_in is None or host_in.shape[0] != batch * n:
                host_in = torch.empty((batch * n, 4), dtype=torch.int64).pin_memory()
                host_out = torch.empty_like(host_in).pin_memory()
                test_host_pipeline_repeated_calls._hin, test_host_pipeline_repeated_calls._hout = host_in, host_out
            host_out = test_host_pipeline_repeated_calls._hout
            host_in.copy_(f.to_ref_layout(x, 64, 4).cpu())
            host_out.zero_()
            plan.host_transform(host_in, host_out, mode="forward", word_bits=64, ref_words=4, chunk=chunk)
            torch.cuda.synchronize()
            assert torch.equal(host_out, want), (batch, chunk)
