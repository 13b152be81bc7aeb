"""Minimal workloads for ncu captures (no CPU baseline, no clocks sampler).

    python tools/workload.py ntt   [--bits 256 --logn 16 --batch 64 --reps 2]
    python tools/workload.py vmul  [--bits 256 --logn 24 --reps 2]
    python tools/workload.py four_step [--bits 256 --logn 24 --reps 2]   (one rank, local exchange)
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["ntt", "vmul", "vadd", "axpy", "four_step"])
    ap.add_argument("--bits", type=int, default=256)
    ap.add_argument("--logn", type=int, default=None)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--strategy", default=None, help="schoolbook/karatsuba (default: the bench's choice)")
    ap.add_argument("--reduction", default="auto", choices=["auto", "barrett"])
    a = ap.parse_args()
    import torch
    from paper_2501_07535_b200 import device as dev
    from paper_2501_07535_b200 import kernels as K
    from paper_2501_07535_b200.params import find_ntt_params
    Kl = (a.bits + 31) // 32

    def rand(count, seed):
        g = torch.Generator(device="cuda").manual_seed(seed)
        x = torch.randint(-(1 << 31), 1 << 31, (count, Kl), dtype=torch.int32, device="cuda", generator=g)
        x[:, Kl - 1] &= (1 << (a.bits - 5 - 32 * (Kl - 1))) - 1
        return x

    if a.what == "ntt":
        logn = a.logn or 16
        prm = find_ntt_params(a.bits, 1 << logn)
        plan = dev.NttPlan(dev.Field(a.bits, prm.p, reduction=a.reduction), prm)
        x = rand(a.batch << logn, 1)
        y = torch.empty_like(x)
        ws = torch.empty(max(1, plan.workspace_bytes(a.batch) // 4), dtype=torch.int32, device="cuda")
        for _ in range(a.reps):
            plan.forward(x, out=y, workspace=ws)
            plan.inverse(y, out=x, workspace=ws)
    elif a.what == "four_step":
        from paper_2501_07535_b200 import dist as D
        logn = a.logn or 24

        class SelfComm:
            def all_to_all(self, out, inp):
                out.copy_(inp)

        eng = D.FourStepNtt(a.bits, find_ntt_params(a.bits, 1 << logn), 0, 1, comm=SelfComm())
        L = eng.layout
        x = rand(L.n1 * L.n2, 1).view(L.n1, L.n2, Kl)
        for _ in range(a.reps):
            eng.forward(x)
    else:
        logn = a.logn or 24
        kara_from = 12 if a.reduction == "auto" else 8  # the bench's choice (bench.py run_blas)
        strat = a.strategy or ("karatsuba" if Kl >= kara_from and a.what != "vadd" else "schoolbook")
        f = dev.Field(a.bits, find_ntt_params(a.bits, 1).p, strat, reduction=a.reduction)
        x, y = rand(1 << logn, 1), rand(1 << logn, 2)
        out = torch.empty_like(x)
        for _ in range(a.reps):
            if a.what == "axpy":
                f.axpy(123456789, x, y, out=out)
            else:
                getattr(f, a.what)(x, y, out=out)
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
