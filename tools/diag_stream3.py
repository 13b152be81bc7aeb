"""Plan creation vs other streams after the suite's three-pass convolve test
(pool blocks freed on the caller's stream) -- which step serialises?"""
import sys, time, gc
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2501_07535_b200 import device as dev
from paper_2501_07535_b200 import kernels as K
from paper_2501_07535_b200.params import find_ntt_params

def trial(label, fn):
    side = torch.cuda.Stream()
    big = torch.empty(1 << 28, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        torch.cuda._sleep(int(2e9))
        big.add_(1)
    b0 = not side.query()
    t0 = time.perf_counter()
    r = fn()
    dt = time.perf_counter() - t0
    busy = not side.query()
    torch.cuda.synchronize()
    print(f"{label:55s} before={b0} busy_after={busy} took={dt*1e3:.1f} ms", flush=True)
    return r

prm = find_ntt_params(128, 1 << 10)
f = dev.Field(128, prm.p)
keep = [trial("baseline plan", lambda: dev.NttPlan(f, prm))]
for bits, logn in [(256, 23), (1024, 19)]:
    plan = K.get_plan(bits, find_ntt_params(bits, 1 << logn))
    n = 1 << logn
    a = torch.zeros((n, plan.limbs), dtype=torch.int32, device="cuda")
    b = torch.zeros_like(a)
    plan.convolve(a, b)
    torch.cuda.synchronize()
    keep.append(trial(f"plan after convolve {bits}/{logn}", lambda: dev.NttPlan(f, prm)))
del a, b
gc.collect()
keep.append(trial("plan after gc", lambda: dev.NttPlan(f, prm)))
x = torch.zeros((1 << 16, 4), dtype=torch.int32, device="cuda")
trial("forward batch 64", lambda: keep[0].forward(x))
trial("field create", lambda: dev.Field(128, prm.p))
