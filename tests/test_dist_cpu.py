"""Multi-process (gloo, world_size 2) coverage of the distributed paths on
CPU: batch sharding, the four-step index maps and the all-to-all block
layout of FourStepNtt.  The rank-local compute is an oracle-backed stand-in
for the device kernels (same interface as dist.DeviceBackend), so the
orchestration — which blocks go where — is checked against the oracle's
full-length transform."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_07535_b200 import dist as D
from paper_2501_07535_b200.params import find_ntt_params


def test_shard_range():
    for total in (0, 1, 7, 64, 256):
        for world in (1, 2, 3, 8):
            parts = [D.shard_range(total, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_split_lengths():
    """Balanced split by default; with the limb count, n >= 2^20 at <= 12 limbs
    puts one 1024-point pass on each phase-1 row (dist.split_lengths)."""
    assert D.split_lengths(1 << 10) == (32, 32)
    assert D.split_lengths(1 << 11) == (64, 32)
    assert D.split_lengths(1 << 24) == (4096, 4096)
    assert D.split_lengths(1 << 24, 8) == (16384, 1024)
    assert D.split_lengths(1 << 20, 12) == (1024, 1024)
    assert D.split_lengths(1 << 24, 24) == (4096, 4096)
    assert D.split_lengths(1 << 16, 8) == (256, 256)
    for n in (1 << 20, 1 << 22, 1 << 24, 1 << 26):
        n1, n2 = D.split_lengths(n, 8)
        assert n1 * n2 == n and n1 >= n2
    with pytest.raises(ValueError):
        D.split_lengths(3)


def test_layout_maps_roundtrip():
    n = 1 << 10
    L = D.FourStepLayout(n, *D.split_lengths(n), 4)
    x = np.arange(n)
    locs = [L.scatter_input(x, r) for r in range(4)]
    assert locs[1][0, 0] == L.n1 // 4  # row j1 = 8, j2 = 0
    assert locs[0][3, 2] == 3 + L.n1 * 2  # x[j1 + N1 j2]
    assert np.array_equal(L.gather_input(locs), x)
    ylocs = [L.scatter_output(x, r) for r in range(4)]
    assert np.array_equal(L.gather_output(ylocs), x)
    with pytest.raises(ValueError):
        D.FourStepLayout(n, 32, 32, 3)


class OracleBackend:
    """CPU stand-in for DeviceBackend (test only): oracle NTT rows, Python-int
    twiddles, numpy transposes."""

    def __init__(self, bits, params, layout, rank):
        from oracle.cbind import OracleField
        self.of = OracleField(params.p, bits)
        self.K = self.of.K
        self.prm, self.L, self.rank = params, layout, rank

    def _np(self, t):
        return t.numpy().view(np.uint32).reshape(-1, self.K)

    def _t(self, a, shape):
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int32).reshape(tuple(shape) + (self.K,)))

    def empty(self, shape):
        return torch.empty(tuple(shape) + (self.K,), dtype=torch.int32)

    def row_ntt(self, x, length, inverse):
        p, w = self.prm.p, self.prm.root
        step = self.prm.n // length
        root = pow(w, step, p)
        if inverse:
            y = self.of.ntt(self._np(x), length, pow(root, -1, p), pow(length, -1, p))
        else:
            y = self.of.ntt(self._np(x), length, root)
        return self._t(y, x.shape[:-1])

    def scale_transpose(self, x, inverse):
        p, n = self.prm.p, self.prm.n
        w = self.prm.root_inv if inverse else self.prm.root
        rows, cols = x.shape[0], x.shape[1]
        row0 = self.rank * rows
        tab = [pow(w, ((row0 + r) * c) % n, p) for r in range(rows) for c in range(cols)]
        tl = np.frombuffer(b"".join(v.to_bytes(4 * self.K, "little") for v in tab), dtype="<u4").reshape(-1, self.K)
        prod = self.of.vector("vmul", self._np(x), np.ascontiguousarray(tl))
        out = np.swapaxes(prod.reshape(rows, cols, self.K), 0, 1)
        return self._t(out, (cols, rows))

    def block_transpose(self, x, rows, cols, block):
        a = self._np(x).reshape(rows, cols, block, self.K)
        return self._t(np.swapaxes(a, 0, 1), (cols, rows * block))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, bits, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prm = find_ntt_params(bits, n)
        layout = D.FourStepLayout(n, *D.split_lengths(n), world)
        be = OracleBackend(bits, prm, layout, rank)
        eng = D.FourStepNtt(bits, prm, rank, world, backend=be, comm=D.TorchComm())
        rng = np.random.Generator(np.random.PCG64(5))
        K = be.K
        xg = rng.integers(0, 1 << 32, size=(n, K), dtype=np.uint64).astype(np.uint32)
        xg[:, -1] &= (1 << 27) - 1
        xl = torch.from_numpy(np.ascontiguousarray(layout.scatter_input(xg, rank)).view(np.int32))
        yl = eng.forward(xl)
        back = eng.inverse(yl)
        result_q.put((rank, yl.numpy().view(np.uint32).copy(), bool(torch.equal(back, xl))))
    finally:
        dist.destroy_process_group()


def test_four_step_gloo_world2():
    n, bits, world = 1 << 10, 256, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, bits, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, _, ok in results), "INTT(NTT(x)) != x across ranks"
    layout = D.FourStepLayout(n, *D.split_lengths(n), world)
    y = layout.gather_output([r[1] for r in results])
    from oracle.cbind import OracleField
    prm = find_ntt_params(bits, n)
    rng = np.random.Generator(np.random.PCG64(5))
    xg = rng.integers(0, 1 << 32, size=(n, 8), dtype=np.uint64).astype(np.uint32)
    xg[:, -1] &= (1 << 27) - 1
    want = OracleField(prm.p, bits).ntt(xg, n, prm.root)
    assert np.array_equal(y, want)
