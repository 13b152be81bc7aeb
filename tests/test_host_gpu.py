"""Host-buffer BLAS (wm_blas_host) and the int <-> limb marshalling of the
drop-in calls: results equal the device-resident kernels and Python ints for
every op, both reference word sizes, ragged lengths and chunkings, and with
the output aliasing an input (reference run_vector, kernels.py:467-480;
to_words/from_words, kernels.py:418-428)."""

from __future__ import annotations

import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rand(torch, n, bits, seed):
    K = (bits + 31) // 32
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randint(-(1 << 31), 1 << 31, (n, K), dtype=torch.int32, device="cuda", generator=g)
    x[:, K - 1] &= (1 << (bits - 5 - 32 * (K - 1))) - 1
    return x


@pytest.mark.parametrize("bits", [128, 256, 384, 768])
@pytest.mark.parametrize("word_bits", [32, 64])
@pytest.mark.parametrize("n,chunk", [(1, 0), (1000, 0), (1000, 7), ((1 << 20) + 3, 0), ((1 << 18) + 1, 50000)])
def test_host_op_matches_device(cuda, bits, word_bits, n, chunk):
    torch = cuda
    from paper_2501_07535_b200 import device as dev
    from paper_2501_07535_b200.params import find_ntt_params
    q = find_ntt_params(bits, 1).p
    f = dev.Field(bits, q)
    a, b = _rand(torch, n, bits, 1 + n), _rand(torch, n, bits, 2 + n)
    P = 1 << ((-(-bits // word_bits)) - 1).bit_length()
    ah = f.to_ref_layout(a, word_bits, P).cpu().pin_memory()
    bh = f.to_ref_layout(b, word_bits, P).cpu().pin_memory()
    oh = torch.empty_like(ah).pin_memory()
    s = 0xDEADBEEF % q
    for kind, want in (("vadd", f.vadd(a, b)), ("vsub", f.vsub(a, b)), ("vmul", f.vmul(a, b)),
                       ("axpy", f.axpy(s, a, b))):
        f.host_op(kind, ah, bh, oh, scalar=s, word_bits=word_bits, ref_words=P, chunk=chunk)
        torch.cuda.synchronize()
        got = f.from_ref_layout(oh.cuda(), word_bits, P)
        assert torch.equal(got, want), kind


def test_host_op_aliasing_and_errors(cuda):
    torch = cuda
    from paper_2501_07535_b200 import device as dev
    from paper_2501_07535_b200.params import find_ntt_params
    q = find_ntt_params(256, 1).p
    f = dev.Field(256, q)
    n = 300001
    a, b = _rand(torch, n, 256, 7), _rand(torch, n, 256, 8)
    ah = f.to_ref_layout(a, 64, 4).cpu().pin_memory()
    bh = f.to_ref_layout(b, 64, 4).cpu().pin_memory()
    f.host_op("vmul", ah, bh, ah, chunk=4096)  # out aliases a
    torch.cuda.synchronize()
    assert torch.equal(f.from_ref_layout(ah.cuda(), 64, 4), f.vmul(a, b))
    with pytest.raises(ValueError):
        f.host_op("axpy", ah, bh, ah, scalar=q)
    with pytest.raises(ValueError):
        f.host_op("vmul", ah, bh[:-4], ah)
    with pytest.raises(ValueError):
        f.host_op("vdiv", ah, bh, ah)


def test_host_ntt_still_matches_after_pipeline_refactor(cuda):
    torch = cuda
    from paper_2501_07535_b200 import kernels as K
    from paper_2501_07535_b200.params import find_ntt_params
    n, batch = 1 << 12, 37
    prm = find_ntt_params(256, n)
    plan = K.get_plan(256, prm)
    x = _rand(torch, n * batch, 256, 9)
    want = plan.forward(x)
    h = plan.field.to_ref_layout(x, 64, 4).cpu().pin_memory()
    o = torch.empty_like(h).pin_memory()
    plan.host_transform(h, o, mode="forward", word_bits=64, ref_words=4, chunk=5)
    torch.cuda.synchronize()
    assert torch.equal(plan.field.from_ref_layout(o.cuda(), 64, 4), want)
