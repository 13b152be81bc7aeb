"""The distributed four-step NTT on the B200: P virtual ranks on one GPU (the
all-to-all as block copies, dist.loopback_transform) with the real device
backend, checked against the single-GPU plan and the oracle; plus the
transpose / twiddle-table kernels it is built from."""

from __future__ import annotations

import random

import numpy as np
import pytest

from oracle.cbind import OracleField

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("logn,P", [(10, 1), (10, 2), (12, 4), (16, 2), (16, 8)])
def test_loopback_four_step_matches_single_gpu(cuda, logn, P):
    import torch
    from paper_2501_07535_b200 import dist as D
    from paper_2501_07535_b200 import kernels as K
    from paper_2501_07535_b200.params import find_ntt_params
    n = 1 << logn
    prm = find_ntt_params(256, n)
    engines = [D.FourStepNtt(256, prm, r, P) for r in range(P)]
    L = engines[0].layout
    g = torch.Generator(device="cuda").manual_seed(logn * 10 + P)
    x = torch.randint(-(1 << 31), 1 << 31, (n, 8), dtype=torch.int32, device="cuda", generator=g)
    x[:, 7] &= (1 << 27) - 1
    xs = [L.scatter_input(x, r) for r in range(P)]
    ys = D.loopback_transform(engines, xs)
    y = L.gather_output([t.cpu().numpy() for t in ys])
    want = K.get_plan(256, prm).forward(x).cpu().numpy()
    assert np.array_equal(y, want)
    back = D.loopback_transform(engines, ys, inverse=True)
    for r in range(P):
        assert torch.equal(back[r], xs[r])


@pytest.mark.parametrize("logn,P", [(10, 1), (12, 4), (16, 2), (16, 8), (20, 16)])
def test_loopback_fused_exchange_matches_nccl_form(cuda, logn, P):
    """The all-to-all fused into the twiddle/transpose kernel (peer stores into
    every rank's receive buffer) gives the same rank-local results as the
    separate exchange, forward and inverse."""
    import torch
    from paper_2501_07535_b200 import dist as D
    from paper_2501_07535_b200.params import find_ntt_params
    n = 1 << logn
    prm = find_ntt_params(256, n)
    engines = [D.FourStepNtt(256, prm, r, P) for r in range(P)]
    L = engines[0].layout
    g = torch.Generator(device="cuda").manual_seed(logn + 100 * P)
    x = torch.randint(-(1 << 31), 1 << 31, (n, 8), dtype=torch.int32, device="cuda", generator=g)
    x[:, 7] &= (1 << 27) - 1
    xs = [L.scatter_input(x, r) for r in range(P)]
    ys = D.loopback_transform(engines, xs)
    yf = D.loopback_transform_fused(engines, xs)
    for a, b in zip(ys, yf):
        assert torch.equal(a, b)
    back = D.loopback_transform_fused(engines, yf, inverse=True)
    for r in range(P):
        assert torch.equal(back[r], xs[r])


def test_loopback_full_width_field(cuda):
    """The distributed four-step over a full-width (Montgomery) field:
    BLS12-381 r at 256 bits, both exchange forms, against the single-GPU plan."""
    import torch
    from paper_2501_07535_b200 import device as dev
    from paper_2501_07535_b200 import dist as D
    from paper_2501_07535_b200.params import NttParams
    r = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001
    n, P = 1 << 16, 4
    w = pow(7, (r - 1) // n, r)
    prm = NttParams(n=n, p=r, root=w, root_inv=pow(w, -1, r), n_inv=pow(n, -1, r))
    engines = [D.FourStepNtt(256, prm, k, P, strategy="montgomery") for k in range(P)]
    L = engines[0].layout
    g = torch.Generator(device="cuda").manual_seed(381)
    x = torch.randint(-(1 << 31), 1 << 31, (n, 8), dtype=torch.int32, device="cuda", generator=g)
    x[:, 7] &= (1 << 28) - 1
    xs = [L.scatter_input(x, k) for k in range(P)]
    ys = D.loopback_transform(engines, xs)
    yf = D.loopback_transform_fused(engines, xs)
    want = dev.NttPlan(dev.Field(256, r, "montgomery"), prm).forward(x).cpu().numpy()
    assert np.array_equal(L.gather_output([t.cpu().numpy() for t in ys]), want)
    for a, b in zip(ys, yf):
        assert torch.equal(a, b)
    back = D.loopback_transform_fused(engines, yf, inverse=True)
    for k in range(P):
        assert torch.equal(back[k], xs[k])


def test_scatter_argument_errors(cuda):
    import torch
    from paper_2501_07535_b200 import _lib
    from paper_2501_07535_b200 import device as dev
    from paper_2501_07535_b200.params import find_ntt_params
    lib = _lib.load()
    f = dev.Field(256, find_ntt_params(256, 1 << 10).p)
    x = torch.zeros((4, 6, 8), dtype=torch.int32, device="cuda")
    t = torch.zeros((4, 6, 16), dtype=torch.int32, device="cuda")
    import ctypes
    st = torch.cuda.current_stream().cuda_stream
    ptrs = (ctypes.c_uint64 * 17)(*([x.data_ptr() + 4096] * 17))
    with pytest.raises(_lib.Unsupported):  # more than 16 peers
        _lib.check(lib.wm_scale_transpose_scatter(f.handle, x.data_ptr(), t.data_ptr(), ptrs, 17, 0, 4, 6, st))
    with pytest.raises(ValueError):  # P does not divide cols
        _lib.check(lib.wm_scale_transpose_scatter(f.handle, x.data_ptr(), t.data_ptr(), ptrs, 4, 0, 4, 6, st))
    with pytest.raises(ValueError):  # source rank out of range
        _lib.check(lib.wm_scale_transpose_scatter(f.handle, x.data_ptr(), t.data_ptr(), ptrs, 2, 2, 4, 6, st))


def test_symmetric_memory_comm_single_rank(cuda):
    """SymmComm plumbing (symmetric-memory rendezvous, peer pointers,
    device barrier) on a one-rank NCCL group: the fused four-step equals the
    single-GPU plan.  Skips where symmetric memory is unavailable."""
    import os
    import torch
    import torch.distributed as dist
    from paper_2501_07535_b200 import dist as D
    from paper_2501_07535_b200 import kernels as K
    from paper_2501_07535_b200.params import find_ntt_params
    if dist.is_initialized():
        pytest.skip("process group already initialised")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29571")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n = 1 << 12
        prm = find_ntt_params(256, n)
        try:
            comm = D.SymmComm(n * 8)
        except Exception as exc:  # no symmetric-memory support in this torch/driver
            pytest.skip(f"symmetric memory unavailable: {exc}")
        eng = D.FourStepNtt(256, prm, 0, 1, comm=comm)
        x = torch.randint(0, 1 << 27, (n, 8), dtype=torch.int32, device="cuda")
        xl = eng.layout.scatter_input(x, 0)
        y = eng.forward(xl)
        want = K.get_plan(256, prm).forward(x).cpu().numpy()
        assert np.array_equal(eng.layout.gather_output([y.cpu().numpy()]), want)
        assert torch.equal(eng.inverse(y), xl)
    finally:
        dist.destroy_process_group()


def test_transpose_kernel(cuda):
    import torch
    from paper_2501_07535_b200 import _lib
    lib = _lib.load()
    for words, rows, cols, batch in [(8, 33, 70, 2), (1, 1, 5, 1), (96, 8, 40, 1), (16, 64, 64, 3)]:
        x = torch.randint(-(1 << 31), 1 << 31, (batch, rows, cols, words), dtype=torch.int32, device="cuda")
        y = torch.empty((batch, cols, rows, words), dtype=torch.int32, device="cuda")
        _lib.check(lib.wm_transpose(words, x.data_ptr(), y.data_ptr(), rows, cols, batch,
                                    torch.cuda.current_stream().cuda_stream))
        assert torch.equal(y, x.transpose(1, 2))


def test_twiddle_table_and_scale_transpose(cuda):
    import torch
    from paper_2501_07535_b200 import _lib
    from paper_2501_07535_b200 import device as dev
    from paper_2501_07535_b200.params import find_ntt_params
    lib = _lib.load()
    n = 1 << 12
    prm = find_ntt_params(256, n)
    f = dev.Field(256, prm.p)
    rows, cols, row0 = 20, 37, 100
    tab = torch.empty((rows, cols, 16), dtype=torch.int32, device="cuda")
    root = _lib.u32_array(dev.ints_to_limbs([prm.root], 8)[0].tolist())
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.wm_twiddle_table_2d(f.handle, n, root, row0, rows, cols, tab.data_ptr(), st))
    got = dev.limbs_to_ints(dev.to_host(tab[..., :8].contiguous()).reshape(-1, 8))
    want = [pow(prm.root, ((row0 + r) * c) % n, prm.p) for r in range(rows) for c in range(cols)]
    assert got == want
    comp = dev.limbs_to_ints(dev.to_host(tab[..., 8:].contiguous()).reshape(-1, 8))
    assert comp == [(w << 256) // prm.p for w in want]
    rnd = random.Random(1)
    xs = [rnd.randrange(prm.p) for _ in range(rows * cols)]
    x = dev.to_device(dev.ints_to_limbs(xs, 8)).reshape(rows, cols, 8)
    out = torch.empty((cols, rows, 8), dtype=torch.int32, device="cuda")
    _lib.check(lib.wm_scale_transpose(f.handle, x.data_ptr(), tab.data_ptr(), out.data_ptr(), rows, cols, st))
    got = dev.limbs_to_ints(dev.to_host(out).reshape(-1, 8))
    exp = [xs[r * cols + c] * want[r * cols + c] % prm.p for c in range(cols) for r in range(rows)]
    assert got == exp


def test_loopback_2p24_roundtrip_and_points(cuda):
    """Config 5 size on one GPU as 2 virtual ranks: roundtrip and random
    output points against the O(n) oracle."""
    import torch
    from paper_2501_07535_b200 import dist as D
    from paper_2501_07535_b200.params import find_ntt_params
    n, P = 1 << 24, 2
    prm = find_ntt_params(256, n)
    engines = [D.FourStepNtt(256, prm, r, P) for r in range(P)]
    L = engines[0].layout
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randint(-(1 << 31), 1 << 31, (n, 8), dtype=torch.int32, device="cuda", generator=g)
    x[:, 7] &= (1 << 27) - 1
    xs = [L.scatter_input(x, r) for r in range(P)]
    ys = D.loopback_transform(engines, xs)
    back = D.loopback_transform(engines, ys, inverse=True)
    for r in range(P):
        assert torch.equal(back[r], xs[r])
    y = L.gather_output([t.cpu().numpy() for t in ys])
    ks = [0, 5, n - 1] + [random.Random(3).randrange(n) for _ in range(3)]
    pts = OracleField(prm.p, 256).ntt_points(x.cpu().numpy().view(np.uint32), prm.root, ks)
    for i, k in enumerate(ks):
        assert np.array_equal(y[k].view(np.uint32), pts[i])


@pytest.mark.parametrize("bits,strategy,logn", [(256, "schoolbook", 12), (256, "barrett", 12), (384, "schoolbook", 11),
                                                (256, "montgomery", 12), (128, "schoolbook", 13)])
def test_factored_twiddles_scale_transpose(cuda, bits, strategy, logn):
    """wm_twiddle_factors + wm_scale_transpose_fx: root^((row0 + r) c) from two
    O(sqrt n) factor tables, times the data, transposed — against Python ints,
    for special-form, Barrett and Montgomery fields; and the fused scatter in
    both layouts (layout 1 = the receiving rank's phase-2 rows)."""
    import torch
    from paper_2501_07535_b200 import _lib
    from paper_2501_07535_b200 import device as dev
    from paper_2501_07535_b200.params import NttParams, find_ntt_params
    lib = _lib.load()
    n = 1 << logn
    if strategy == "montgomery":
        p = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001
        w = pow(7, (p - 1) // n, p)
        prm = NttParams(n=n, p=p, root=w, root_inv=pow(w, -1, p), n_inv=pow(n, -1, p))
        f = dev.Field(bits, p, "montgomery")
    else:
        prm = find_ntt_params(bits, n)
        f = dev.Field(bits, prm.p, reduction="barrett" if strategy == "barrett" else "auto")
    K = f.limbs
    logB = (logn + 1) // 2
    lo = torch.empty((1 << logB, K), dtype=torch.int32, device="cuda")
    hi = torch.empty((n >> logB, K), dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    root = _lib.u32_array(dev.ints_to_limbs([prm.root], K)[0].tolist())
    _lib.check(lib.wm_twiddle_factors(f.handle, n, root, logB, lo.data_ptr(), hi.data_ptr(), st))
    rows, cols, row0, P = 24, 40, 17, 4
    rnd = random.Random(logn + bits)
    xs = [rnd.randrange(prm.p) for _ in range(rows * cols)]
    xs[:cols] = [prm.p - 1] * cols
    x = dev.to_device(dev.ints_to_limbs(xs, K)).reshape(rows, cols, K)
    want = [xs[r * cols + c] * pow(prm.root, ((row0 + r) * c) % n, prm.p) % prm.p
            for c in range(cols) for r in range(rows)]
    out = torch.empty((cols, rows, K), dtype=torch.int32, device="cuda")
    _lib.check(lib.wm_scale_transpose_fx(f.handle, x.data_ptr(), lo.data_ptr(), hi.data_ptr(), logB, n, row0,
                                         out.data_ptr(), None, 0, 0, 0, rows, cols, st))
    assert dev.limbs_to_ints(dev.to_host(out).reshape(-1, K)) == want
    import ctypes
    for layout in (0, 1):
        recv = [torch.zeros((P, cols // P, rows, K), dtype=torch.int32, device="cuda") for _ in range(P)]
        arr = (ctypes.c_uint64 * P)(*[t.data_ptr() for t in recv])
        src = 2
        _lib.check(lib.wm_scale_transpose_fx(f.handle, x.data_ptr(), lo.data_ptr(), hi.data_ptr(), logB, n, row0,
                                             None, arr, P, src, layout, rows, cols, st))
        for d in range(P):
            block = out[d * (cols // P):(d + 1) * (cols // P)]  # [cols/P][rows][K]
            if layout == 0:
                assert torch.equal(recv[d][src], block)
            else:  # [cols/P][P * rows]: source src's rows at columns src*rows ..
                got = recv[d].reshape(cols // P, P, rows, K)[:, src]
                assert torch.equal(got, block)
