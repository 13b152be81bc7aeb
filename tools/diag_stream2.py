"""Plan creation vs other streams, after the pool has freed memory and with
the default mempool's release threshold raised (which step serialises?)."""
import ctypes, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2501_07535_b200 import device as dev
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
    print(f"{label:50s} busy_after={busy} took={dt*1e3:.1f} ms", flush=True)
    return r

torch.cuda._sleep(1000); torch.cuda.synchronize()
prm = find_ntt_params(128, 1 << 10)
trial("warm-up sleep only", lambda: None)
f0 = dev.Field(128, prm.p)
p0 = dev.NttPlan(f0, prm); torch.cuda.synchronize(); del p0  # pool now holds freed memory
f1 = dev.Field(128, prm.p)
p1 = trial("A: plan after a destroyed plan (same K)", lambda: dev.NttPlan(f1, prm))
prm12 = find_ntt_params(384, 1 << 10)
f12 = dev.Field(384, prm12.p)  # preloads K=12 kernels
p12 = trial("C: plan of a new K after its field preloaded", lambda: dev.NttPlan(f12, prm12))
p12b = trial("C2: second plan of that K", lambda: dev.NttPlan(f12, prm12))
x = torch.zeros((1 << 10, 12), dtype=torch.int32, device="cuda")
trial("C3: first forward of that K", lambda: p12.forward(x))
cudart = ctypes.CDLL(str(Path(torch.__file__).parent.parent / "nvidia/cuda_runtime/lib/libcudart.so.12"))
pool = ctypes.c_void_p()
print("getpool", cudart.cudaDeviceGetDefaultMemPool(ctypes.byref(pool), 0))
val = ctypes.c_uint64(2**63)
print("setattr", cudart.cudaMemPoolSetAttribute(pool, 4, ctypes.byref(val)))
del p1; torch.cuda.synchronize()
f2 = dev.Field(128, prm.p)
trial("B: plan after a destroyed plan, release threshold max", lambda: dev.NttPlan(f2, prm))
prm16 = find_ntt_params(512, 1 << 10)
f16 = dev.Field(512, prm16.p)
trial("D: new K=16 plan, threshold max (pool growth)", lambda: dev.NttPlan(f16, prm16))
