"""Multi-GPU partitioning of the hot path.

* Batches of independent transforms and BLAS vectors shard by rank with no
  collective at all (``shard_range``): every rank runs its own slice through
  the single-GPU kernels; timing is max-over-ranks (bench.py).
* A single long transform (config 5: 256-bit n = 2^24) is split four-step,
  n = N1 * N2, over P ranks with exactly one all-to-all (``FourStepNtt``):

      rank r holds rows j1 in its block (N1/P rows), row j1 = x[j1 + N1 j2]
      (a) N2-point row NTTs                        wm_ntt_forward
      (b) * root^(j1 k2), transpose to [k2][j1]    wm_scale_transpose_fx (twiddles from two
                                                   O(sqrt n) factor tables, fused)
      (c) all-to-all of the P column blocks        torch.distributed (NCCL)
      (d) [P][N2/P][N1/P] -> [N2/P][N1]            wm_transpose (block transpose)
      (fused exchange: (b)+(c)+(d) are one kernel storing rank d's phase-2
       rows straight into its symmetric-memory receive buffer, SymmComm)
      (e) N1-point row NTTs                        wm_ntt_forward
      rank r now holds rows k2 in its block, row k2 = y[k2 + N2 k1]

  The inverse runs the same five steps with the roles of N1 and N2 swapped
  and inverse roots, mapping the output distribution back to the input one,
  so INTT(NTT(x)) round-trips rank-locally.  The index algebra is the
  four-step factorisation of the reference DFT y[k] = sum_j x[j] root^(jk)
  (ntt_reference, oracle.py:262-282); the reference itself has no multi-GPU
  path.

The local compute is a *backend* object so the orchestration (block layout
of the all-to-all, index maps) can be exercised on CPU with gloo in tests;
the product backend is ``DeviceBackend`` (sm_100a kernels via the C ABI).
"""

from __future__ import annotations

from dataclasses import dataclass

from .params import NttParams


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, stop) slice of `total` items for `rank` (weak or
    strong scaling of batched transforms / BLAS vectors: no collective)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def split_lengths(n: int, limbs: int | None = None) -> tuple[int, int]:
    """n = N1 * N2 with N1 >= N2, both powers of two.

    Balanced (N1 = 2^ceil(log n / 2)) unless the limb count is given: for
    n >= 2^20 at <= 12 limbs the phase-1 rows are one 1024-point pass (the
    most efficient pass length at these widths: 7.7 ps per butterfly in the
    2^20 plan against 8.2 for 256-point passes) and N1 = n / 1024.  At
    256-bit 2^24 that split (2^14 x 2^10) runs 1.2-1.8 % faster than
    2^12 x 2^12 at one rank; a 2^11-point single pass is 7 % slower
    (profiles/r02_ab_four_step_split.txt, r02_fourstep_rerun.txt)."""
    if n < 4 or n & (n - 1):
        raise ValueError("four-step needs a power-of-two length >= 4")
    logn = n.bit_length() - 1
    if limbs is not None and limbs <= 12 and logn >= 20:
        return n >> 10, 1 << 10
    n1 = 1 << ((logn + 1) // 2)
    return n1, n // n1


@dataclass(frozen=True)
class FourStepLayout:
    """Index maps between the global vector and rank-local rows."""

    n: int
    n1: int
    n2: int
    world: int

    def __post_init__(self):
        if self.n1 * self.n2 != self.n:
            raise ValueError("n != N1 * N2")
        if self.n1 % self.world or self.n2 % self.world:
            raise ValueError(f"world size {self.world} must divide N1={self.n1} and N2={self.n2}")

    def input_rows(self, rank: int) -> range:
        b = self.n1 // self.world
        return range(rank * b, (rank + 1) * b)

    def output_rows(self, rank: int) -> range:
        b = self.n2 // self.world
        return range(rank * b, (rank + 1) * b)

    def scatter_input(self, x, rank: int):
        """Global x[n] (array-like with a leading element axis) -> rank-local
        [N1/P, N2, ...]: row j1 = x[j1 + N1*j2]."""
        v = x.reshape((self.n2, self.n1) + tuple(x.shape[1:]))
        r = self.input_rows(rank)
        return _swap01(v[:, r.start:r.stop])

    def gather_output(self, locals_):
        """Rank-local outputs [N2/P, N1, ...] (rank order) -> global y[n]."""
        import numpy as np
        rows = np.concatenate([np.asarray(l) for l in locals_], axis=0)  # [N2, N1, ...]
        return _swap01(rows).reshape((self.n,) + rows.shape[2:])

    def scatter_output(self, y, rank: int):
        v = y.reshape((self.n1, self.n2) + tuple(y.shape[1:]))
        r = self.output_rows(rank)
        return _swap01(v[:, r.start:r.stop])

    def gather_input(self, locals_):
        import numpy as np
        rows = np.concatenate([np.asarray(l) for l in locals_], axis=0)  # [N1, N2, ...]
        return _swap01(rows).reshape((self.n,) + rows.shape[2:])


def _swap01(a):
    import numpy as np
    if isinstance(a, np.ndarray):
        return np.ascontiguousarray(np.swapaxes(a, 0, 1))
    return a.transpose(0, 1).contiguous()


class TorchComm:
    """all-to-all over a torch.distributed process group (NCCL on GPUs)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_to_all(self, out, inp):
        self.dist.all_to_all_single(out.view(-1), inp.view(-1), group=self.group)
        return out


class StagedComm:
    """all-to-all staged through host memory over a CPU process group (gloo):
    the functional stand-in for TorchComm where NCCL cannot run, i.e. several
    ranks sharing one GPU (2-process tests, ``bench.py --dist-backend gloo``
    dry runs).  Same block layout as TorchComm; not a performance path."""

    fused = False

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_to_all(self, out, inp):
        import torch
        torch.cuda.current_stream().synchronize()
        src = inp.reshape(-1).cpu()
        dst = torch.empty_like(src)
        self.dist.all_to_all_single(dst, src, group=self.group)
        out.view(-1).copy_(dst)
        return out


class SymmComm:
    """Peer-memory exchange for the four-step (the all-to-all fused into the
    twiddle/transpose kernel).  Every rank's receive buffer is allocated from
    torch symmetric memory and rendezvoused, so each rank holds the NVLink
    (peer-mapped) addresses of all receive buffers; the producing kernel
    stores each column block straight into its destination rank's buffer and
    a device-side barrier (stream-ordered) publishes the writes.  A barrier
    before the stores keeps a fast rank from overwriting a buffer its peer is
    still reading from the previous call."""

    fused = True

    def __init__(self, n_words: int, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.dist = dist
        self.group = group if group is not None else dist.group.WORLD
        self.rank = dist.get_rank(self.group)
        self.world = dist.get_world_size(self.group)
        dev = torch.device("cuda", torch.cuda.current_device())
        # the local allocation can fail on one rank only; agree before the
        # collective rendezvous so no rank is left waiting in it
        err = None
        try:
            self.recv = symm.empty(n_words, dtype=torch.int32, device=dev)
        except Exception as exc:  # noqa: BLE001 - reported after the agreement
            err = exc
        ok = torch.tensor([0 if err is None else 1], dtype=torch.int32, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MAX, group=self.group)
        if int(ok.item()):
            raise RuntimeError(f"symmetric memory allocation failed on some rank: {err}")
        self.handle = symm.rendezvous(self.recv, self.group.group_name)
        self.peer_ptrs = [int(p) for p in self.handle.buffer_ptrs]
        if len(self.peer_ptrs) != self.world:
            raise RuntimeError("symmetric memory rendezvous returned a wrong peer count")

    def barrier(self):
        self.handle.barrier(channel=0)


class DeviceBackend:
    """Rank-local compute on the B200 (C ABI kernels)."""

    def __init__(self, bits: int, params: NttParams, layout: FourStepLayout, rank: int,
                 strategy: str = "schoolbook"):
        import torch

        from .device import Field, NttPlan, ints_to_limbs
        from . import _lib
        self.torch = torch
        self.layout = layout
        p, n = params.p, params.n
        w, wi = params.root, params.root_inv
        n1, n2, P = layout.n1, layout.n2, layout.world
        self.field = Field(bits, p, strategy)  # "montgomery" for full-width primes
        K = self.field.limbs
        self.K = K

        def sub_params(m: int, step: int) -> NttParams:
            r = pow(w, step, p)
            return NttParams(n=m, p=p, root=r, root_inv=pow(r, -1, p), n_inv=pow(m, -1, p))

        self.plan_n2 = NttPlan(self.field, sub_params(n2, n1))  # root^(N1): order N2
        self.plan_n1 = NttPlan(self.field, sub_params(n1, n2))  # root^(N2): order N1
        lib = self.field.lib
        enc = lambda v: _lib.u32_array(ints_to_limbs([v], K)[0].tolist())  # noqa: E731
        stream = torch.cuda.current_stream().cuda_stream
        # inter-rank twiddles root^(j1 k2) from two factor tables of O(sqrt n)
        # entries (wm_twiddle_factors): 2 x 2^12 entries at n = 2^24
        logn = n.bit_length() - 1
        self.logB = (logn + 1) // 2
        self.rows_f, self.rows_i = n1 // P, n2 // P
        self.row0_f, self.row0_i = rank * self.rows_f, rank * self.rows_i
        self.tw = {}
        for inv, root in ((False, w), (True, wi)):
            lo = torch.empty((1 << self.logB, K), dtype=torch.int32, device="cuda")
            hi = torch.empty((n >> self.logB, K), dtype=torch.int32, device="cuda")
            _lib.check(lib.wm_twiddle_factors(self.field.handle, n, enc(root), self.logB, lo.data_ptr(),
                                              hi.data_ptr(), stream), "wm_twiddle_factors")
            self.tw[inv] = (lo, hi)
        self.n = n
        self.lib = lib
        self._lib = _lib

    def table_bytes(self) -> int:
        """Device bytes of the inter-rank twiddle tables (both directions)."""
        return sum(t.numel() * t.element_size() for pair in self.tw.values() for t in pair)

    def empty(self, shape):
        return self.torch.empty(tuple(shape) + (self.K,), dtype=self.torch.int32, device="cuda")

    def row_ntt(self, x, length: int, inverse: bool):
        plan = self.plan_n2 if length == self.layout.n2 else self.plan_n1
        return plan.inverse(x) if inverse else plan.forward(x)

    def _fx(self, x, inverse: bool, out=None, dst_ptrs=None, src_rank: int = 0, layout: int = 1):
        import ctypes
        rows, cols = x.shape[0], x.shape[1]
        lo, hi = self.tw[inverse]
        row0 = self.row0_i if inverse else self.row0_f
        P = 0 if dst_ptrs is None else len(dst_ptrs)
        arr = None if dst_ptrs is None else (ctypes.c_uint64 * P)(*[int(p) for p in dst_ptrs])
        stream = self.torch.cuda.current_stream().cuda_stream
        self._lib.check(self.lib.wm_scale_transpose_fx(self.field.handle, x.data_ptr(), lo.data_ptr(), hi.data_ptr(),
                                                       self.logB, self.n, row0,
                                                       out.data_ptr() if out is not None else None, arr, P, src_rank,
                                                       layout, rows, cols, stream), "wm_scale_transpose_fx")

    def scale_transpose(self, x, inverse: bool):
        """[rows][cols] -> [cols][rows] times root^((row0 + r) c) (wm_scale_transpose_fx)."""
        out = self.empty((x.shape[1], x.shape[0]))
        self._fx(x, inverse, out=out)
        return out

    def scale_transpose_scatter(self, x, inverse: bool, dst_ptrs, src_rank: int, layout: int = 1):
        """scale_transpose with the all-to-all fused in: column block d of the
        transposed output goes straight into dst_ptrs[d] (rank d's receive
        buffer).  layout 1 stores it as rank d's phase-2 rows
        ([cols/P][P * rows]: no block transpose after the exchange); layout 0
        as an all-to-all's blocks ([P][cols/P][rows])."""
        self._fx(x, inverse, dst_ptrs=dst_ptrs, src_rank=src_rank, layout=layout)

    def block_transpose(self, x, rows: int, cols: int, block: int):
        """[rows][cols][block] -> [cols][rows][block] (block = elements)."""
        out = self.empty((cols, rows * block))
        stream = self.torch.cuda.current_stream().cuda_stream
        self._lib.check(self.lib.wm_transpose(self.K * block, x.data_ptr(), out.data_ptr(), rows, cols, 1,
                                              stream), "wm_transpose")
        return out


class FourStepNtt:
    """One length-n NTT across the ranks of a communicator (see module doc)."""

    def __init__(self, bits: int, params: NttParams, rank: int, world: int, backend=None, comm=None,
                 strategy: str = "schoolbook", split: tuple[int, int] | None = None):
        self.params = params
        if split is None:
            split = split_lengths(params.n, -(-bits // 32))
        self.layout = FourStepLayout(params.n, *split, world)
        self.rank, self.world = rank, world
        self.backend = (backend if backend is not None
                        else DeviceBackend(bits, params, self.layout, rank, strategy))
        self.comm = comm

    # phase 1: local row transforms + twiddle/transpose -> send buffer
    def phase1(self, x, inverse: bool):
        L = self.layout
        row_len = L.n1 if inverse else L.n2
        y = self.backend.row_ntt(x, row_len, inverse)
        return self.backend.scale_transpose(y, inverse)  # [row_len][rows_local]

    # phase 2: received [P][row_len/P][rows_local] -> block transpose -> row transforms
    # (rows=True: received already as rows [row_len/P][other], fused layout 1)
    def phase2(self, d, inverse: bool, rows: bool = False):
        L = self.layout
        P = self.world
        row_len = L.n1 if inverse else L.n2      # length of the phase-1 rows
        other = L.n2 if inverse else L.n1        # length of the phase-2 rows
        rows_local = other // P
        if rows:
            e = d.reshape(row_len // P, other, -1)
        else:
            e = self.backend.block_transpose(d, P, row_len // P, rows_local)  # [row_len/P][other]
        return self.backend.row_ntt(e, other, inverse)

    def _run(self, x, inverse: bool):
        if getattr(self.comm, "fused", False):
            return self._run_fused(x, inverse)
        c = self.phase1(x, inverse)
        d = self.backend.empty(c.shape[:-1]) if hasattr(self.backend, "empty") else c.clone()
        self.comm.all_to_all(d, c)
        return self.phase2(d, inverse)

    def _run_fused(self, x, inverse: bool):
        """Row NTTs, then one kernel that twiddles, transposes and stores every
        column block into its destination rank's receive buffer (NVLink peer
        stores), then the rank-local phase 2 on the received blocks."""
        L = self.layout
        P = self.world
        row_len = L.n1 if inverse else L.n2
        other = L.n2 if inverse else L.n1
        y = self.backend.row_ntt(x, row_len, inverse)
        k = self.backend.K
        words = row_len * (other // P) * k
        self.comm.barrier()  # every peer is done reading its receive buffer
        self.backend.scale_transpose_scatter(y, inverse, self.comm.peer_ptrs, self.rank, layout=1)
        self.comm.barrier()  # every block has landed, as this rank's phase-2 rows
        d = self.comm.recv[:words].view(row_len // P, other, k)
        return self.phase2(d, inverse, rows=True)

    def forward(self, x):
        """x: [N1/P, N2, K] local rows -> [N2/P, N1, K] (rows k2 of y)."""
        return self._run(x, False)

    def inverse(self, y):
        """y: [N2/P, N1, K] -> [N1/P, N2, K] (rows j1 of x)."""
        return self._run(y, True)


def loopback_transform_fused(engines, xs, inverse: bool = False):
    """The fused exchange over P virtual ranks on one GPU: every virtual rank's
    receive buffer is a local tensor and the scatter kernel writes into all of
    them (on a multi-GPU box the same kernel gets peer-mapped addresses)."""
    import torch
    P = len(engines)
    L = engines[0].layout
    row_len = L.n1 if inverse else L.n2
    other = L.n2 if inverse else L.n1
    k = engines[0].backend.K
    recvs = [torch.empty((row_len // P, other, k), dtype=torch.int32, device="cuda") for _ in range(P)]
    ptrs = [r.data_ptr() for r in recvs]
    for r, (e, x) in enumerate(zip(engines, xs)):
        y = e.backend.row_ntt(x, row_len, inverse)
        e.backend.scale_transpose_scatter(y, inverse, ptrs, r, layout=1)
    return [e.phase2(d, inverse, rows=True) for e, d in zip(engines, recvs)]


def loopback_transform(engines, xs, inverse: bool = False):
    """Run a FourStepNtt over P *virtual* ranks in one process (one engine per
    virtual rank, typically all on one GPU): phase 1 on every rank, the
    all-to-all as block copies, phase 2 on every rank.  Used to test the
    distributed algorithm end to end on a single device."""
    P = len(engines)
    sends = [e.phase1(x, inverse) for e, x in zip(engines, xs)]
    rows = sends[0].shape[0] // P  # send buffers are [row_len][rows_local]: P row blocks
    recvs = []
    for r in range(P):
        parts = [s[r * rows:(r + 1) * rows] for s in sends]  # block r of every source, source order
        import torch
        recvs.append(torch.cat([p.reshape(-1) for p in parts]).reshape(sends[0].shape).contiguous())
    return [e.phase2(d, inverse) for e, d in zip(engines, recvs)]
