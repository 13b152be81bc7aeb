"""Edge behaviour of the C ABI on the B200 (round-1 review items): three-pass
convolution, batches beyond one grid dimension, the plan's shared workspace
used from two streams, transposes of more than 65535 rows, non-canonical axpy
scalars and power-of-two moduli rejected, reference-launcher status."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _plan(bits, n):
    from paper_2501_07535_b200 import kernels as K
    from paper_2501_07535_b200.params import find_ntt_params
    return K.get_plan(bits, find_ntt_params(bits, n))


def _rand(torch, rows, K, bits, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randint(-(1 << 31), 1 << 31, (rows, K), dtype=torch.int32, device="cuda", generator=g)
    x[:, K - 1] &= (1 << (bits - 5 - 32 * (K - 1))) - 1  # < 2^(bits-5) < p
    return x


@pytest.mark.parametrize("bits,logn", [(256, 23), (1024, 19)])
def test_convolve_three_pass_plans(cuda, bits, logn):
    """wm_ntt_convolve on three-pass plans equals the unfused sequence
    INTT(NTT(a) * NTT(b)) (forward, vmul, inverse as separate calls), and is
    symmetric in a, b; a may alias out."""
    torch = cuda
    n = 1 << logn
    plan = _plan(bits, n)
    assert len(plan.pass_log_sizes) == 3
    K = plan.limbs
    a = _rand(torch, n, K, bits, 1)
    b = _rand(torch, n, K, bits, 2)
    want = plan.inverse(plan.field.vmul(plan.forward(a), plan.forward(b)))
    got = plan.convolve(a, b)
    assert torch.equal(got, want)
    assert torch.equal(plan.convolve(b, a), want)
    a2 = a.clone()
    plan.convolve(a2, b, out=a2)
    assert torch.equal(a2, want)


def test_multi_pass_batch_above_65535(cuda):
    """A two-pass plan over 65537 transforms (grid.y chunking) equals the same
    transforms run in two calls."""
    torch = cuda
    n, batch = 1 << 12, 65537
    plan = _plan(32, n)
    assert len(plan.pass_log_sizes) == 2
    x = _rand(torch, batch * n, plan.limbs, 32, 3)
    y = plan.forward(x)
    head = plan.forward(x[: 65536 * n].contiguous())
    tail = plan.forward(x[65536 * n:].contiguous())
    assert torch.equal(y[: 65536 * n], head)
    assert torch.equal(y[65536 * n:], tail)
    assert torch.equal(plan.inverse(y), x)


def test_plan_workspace_from_two_streams(cuda):
    """Multi-pass calls without a workspace on two streams at once share the
    plan's workspace; its uses are stream-ordered, so both results are exact."""
    torch = cuda
    n, batch = 1 << 16, 16
    plan = _plan(256, n)
    xs = [_rand(torch, batch * n, 8, 256, 10 + i) for i in range(2)]
    want = [plan.forward(x) for x in xs]
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = [torch.empty_like(x) for x in xs]
    for _ in range(3):
        for o in outs:
            o.zero_()
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            plan.forward(xs[0], out=outs[0], stream=s1)
        with torch.cuda.stream(s2):
            plan.forward(xs[1], out=outs[1], stream=s2)
        torch.cuda.synchronize()
        assert torch.equal(outs[0], want[0]) and torch.equal(outs[1], want[1])


@pytest.mark.parametrize("words,rows,cols,batch", [(8, 70000, 3, 1), (64, 66000, 2, 2), (3, 5, 7, 70000)])
def test_transpose_large_grids(cuda, words, rows, cols, batch):
    torch = cuda
    from paper_2501_07535_b200 import _lib
    lib = _lib.load()
    x = torch.randint(-(1 << 31), 1 << 31, (batch, rows, cols, words), dtype=torch.int32, device="cuda")
    out = torch.empty_like(x)
    _lib.check(lib.wm_transpose(words, x.data_ptr(), out.data_ptr(), rows, cols, batch,
                                torch.cuda.current_stream().cuda_stream))
    assert torch.equal(out.view(batch, cols, rows, words), x.transpose(1, 2))


def test_axpy_scalar_must_be_canonical(cuda):
    torch = cuda
    from paper_2501_07535_b200 import _lib
    from paper_2501_07535_b200 import device as dev
    from paper_2501_07535_b200.params import find_ntt_params
    q = find_ntt_params(256, 1).p
    f = dev.Field(256, q)
    x = _rand(torch, 64, 8, 256, 5)
    with pytest.raises(ValueError):
        f.axpy(q, x, x)
    with pytest.raises(ValueError):
        f.axpy(-1, x, x)
    # the C ABI itself rejects it too (no silent wrong answers for direct callers)
    lib = _lib.load()
    s = _lib.u32_array(dev.ints_to_limbs([q + 5], 8)[0].tolist())
    rc = lib.wm_axpy(f.handle, s, x.data_ptr(), x.data_ptr(), x.data_ptr(), 64, None)
    assert rc == _lib.WM_EINVAL
    assert f.axpy(q - 1, x, x).shape == x.shape


def test_power_of_two_modulus_rejected(cuda):
    from paper_2501_07535_b200 import _lib
    from paper_2501_07535_b200 import device as dev
    for bits, q in [(32, 1 << 27), (64, 1 << 40), (256, 1 << 251)]:
        with pytest.raises(ValueError):
            dev.Field(bits, q)


def test_plan_creation_leaves_other_streams_running(cuda):
    """Plan creation uses a private stream: work queued on another stream is
    not forced to complete (no device-wide synchronisation).  A long kernel
    is queued on a side stream, then a plan is created; the side stream must
    still be busy when creation returns."""
    torch = cuda
    from paper_2501_07535_b200 import device as dev
    from paper_2501_07535_b200.params import find_ntt_params
    # the field loads its kernel images (CUDA lazy loading synchronises the
    # context on a kernel's first load), so it is created before the side work
    prm = find_ntt_params(128, 1 << 10)
    field = dev.Field(128, prm.p)
    import gc
    gc.collect()
    side = torch.cuda.Stream()
    big = torch.empty(1 << 28, dtype=torch.int32, device="cuda")
    # torch's own kernels load lazily too: the first launch of the side work's
    # kernels would synchronise the context right here (before plan creation),
    # so run them once first
    with torch.cuda.stream(side):
        torch.cuda._sleep(1000)
        big.add_(1)
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        torch.cuda._sleep(int(2e9))  # ~1 s of GPU clock cycles
        big.add_(1)
    # keep the plan alive past the check: destroying it frees device memory
    # (cudaFree synchronises the device by definition).  Earlier tests' plans
    # and fields still waiting for the garbage collector would do the same if
    # a collection ran inside the measured call, so collect first and keep
    # the collector off while measuring.
    import gc
    gc.collect()
    gc.disable()
    import time
    try:
        busy_before = not side.query()
        t0 = time.perf_counter()
        plan = dev.NttPlan(field, prm)
        took = time.perf_counter() - t0
        busy = not side.query()
    finally:
        gc.enable()
    torch.cuda.synchronize()
    del plan
    assert busy, (f"plan creation waited for an unrelated stream (side busy before: {busy_before}, "
                  f"creation took {took * 1e3:.1f} ms)")
    side.synchronize()
