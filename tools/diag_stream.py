"""Which step of plan creation waits for other streams?  A long kernel is
queued on a side stream; after each step we ask whether it is still busy."""
import ctypes, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2501_07535_b200 import device as dev, _lib
from paper_2501_07535_b200.params import find_ntt_params

def trial(label, fn):
    side = torch.cuda.Stream()
    big = torch.empty(1 << 28, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        torch.cuda._sleep(int(2e9))
        big.add_(1)
    t0 = time.perf_counter()
    r = fn()
    dt = time.perf_counter() - t0
    busy = not side.query()
    torch.cuda.synchronize()
    print(f"{label:40s} busy_after={busy} took={dt*1e3:.1f} ms", flush=True)
    return r

prm = find_ntt_params(128, 1 << 10)
f = trial("field create", lambda: dev.Field(128, prm.p))
p1 = trial("plan create (1st, cold kernels)", lambda: dev.NttPlan(f, prm))
p2 = trial("plan create (2nd, warm)", lambda: dev.NttPlan(f, prm))
prm2 = find_ntt_params(256, 1 << 12)
f2 = dev.Field(256, prm2.p)
p3 = trial("plan create 256-bit (cold K=8 gen)", lambda: dev.NttPlan(f2, prm2))
p4 = trial("plan create 256-bit (warm)", lambda: dev.NttPlan(f2, prm2))
x = torch.zeros((1 << 12, 8), dtype=torch.int32, device="cuda")
trial("forward (warm)", lambda: p4.forward(x))
