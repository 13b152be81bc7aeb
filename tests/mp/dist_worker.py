"""Worker of tests/test_dist_mp_gpu.py: the real DeviceBackend four-step NTT,
batch-sharded NTTs and rank-sharded BLAS in a 2-process gloo job whose ranks
share one GPU (the all-to-all staged through host memory, dist.StagedComm),
each rank's results checked against the single-GPU plan over the whole
input.  Run under torch.distributed.run."""

from __future__ import annotations

import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main() -> int:
    import torch
    import torch.distributed as dist

    from paper_2501_07535_b200 import device as dev
    from paper_2501_07535_b200 import dist as D
    from paper_2501_07535_b200 import kernels as K
    from paper_2501_07535_b200.params import find_ntt_params

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())

    def rand(count, seed):
        g = torch.Generator(device="cuda").manual_seed(seed)
        x = torch.randint(-(1 << 31), 1 << 31, (count, 8), dtype=torch.int32, device="cuda", generator=g)
        x[:, 7] &= (1 << 27) - 1
        return x

    # (1) single long transforms, four-step over the ranks (one all-to-all)
    for logn in (16, 20):
        n = 1 << logn
        prm = find_ntt_params(256, n)
        eng = D.FourStepNtt(256, prm, rank, world, comm=D.StagedComm())
        L = eng.layout
        x = rand(n, 1000 + logn)  # the same global vector on every rank
        y = eng.forward(L.scatter_input(x, rank))
        want = K.get_plan(256, prm).forward(x)
        assert torch.equal(y, L.scatter_output(want, rank)), f"four-step 2^{logn} forward mismatch"
        back = eng.inverse(y)
        assert torch.equal(back, L.scatter_input(x, rank)), f"four-step 2^{logn} roundtrip mismatch"

    # (2) batched transforms sharded by rank (no collective)
    n, total = 1 << 12, 10
    prm = find_ntt_params(256, n)
    plan = K.get_plan(256, prm)
    xb = rand(total * n, 77).view(total, n, 8)
    lo, hi = D.shard_range(total, rank, world)
    mine = plan.forward(xb[lo:hi].contiguous())
    assert torch.equal(mine, plan.forward(xb)[lo:hi]), "batched shard mismatch"

    # (3) BLAS sharded by rank, gathered on every rank (parity only)
    m = 1 << 16
    f = dev.Field(256, find_ntt_params(256, 1).p)
    a, b = rand(m, 5), rand(m, 6)
    lo, hi = D.shard_range(m, rank, world)
    part = f.vmul(a[lo:hi].contiguous(), b[lo:hi].contiguous()).cpu()
    parts = [None] * world
    dist.all_gather_object(parts, part)
    assert torch.equal(torch.cat(parts), f.vmul(a, b).cpu()), "sharded vmul mismatch"

    dist.barrier()
    print(f"RANK {rank} OK", flush=True)
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
