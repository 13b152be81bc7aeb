"""Which step of NTT plan creation ends a busy side stream early / waits for it?"""
import ctypes, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2501_07535_b200 import device as dev
from paper_2501_07535_b200.params import find_ntt_params

cudart = ctypes.CDLL(str(Path(torch.__file__).parent.parent / "nvidia/cuda_runtime/lib/libcudart.so.12"))
big = torch.empty(1 << 28, dtype=torch.int32, device="cuda")

def trial(label, fn):
    side = torch.cuda.Stream()
    torch.cuda.synchronize()
    t00 = time.perf_counter()
    with torch.cuda.stream(side):
        torch.cuda._sleep(int(2e9))
        big.add_(1)
    b0 = not side.query()
    t0 = time.perf_counter()
    r = fn()
    dt = time.perf_counter() - t0
    busy = not side.query()
    t1 = time.perf_counter()
    side.synchronize()
    rest = time.perf_counter() - t1
    print(f"{label:45s} before={b0} busy_after={busy} took={dt*1e3:.1f} ms side_rest={rest*1e3:.0f} ms "
          f"side_total={(time.perf_counter()-t00)*1e3:.0f} ms", flush=True)
    return r

def stream_cd():
    s = ctypes.c_void_p()
    cudart.cudaStreamCreateWithFlags(ctypes.byref(s), 1)
    cudart.cudaStreamDestroy(s)

def malloc_async():
    s = ctypes.c_void_p(); p = ctypes.c_void_p()
    cudart.cudaStreamCreateWithFlags(ctypes.byref(s), 1)
    cudart.cudaMallocAsync(ctypes.byref(p), ctypes.c_size_t(1 << 20), s)
    cudart.cudaFreeAsync(p, s)
    cudart.cudaStreamSynchronize(s)
    cudart.cudaStreamDestroy(s)

trial("nothing", lambda: time.sleep(0.001))
trial("stream create/destroy", stream_cd)
trial("mallocAsync on private stream", malloc_async)
prm = find_ntt_params(128, 1 << 10)
f = trial("field create 128", lambda: dev.Field(128, prm.p))
p1 = trial("plan create 128 (first)", lambda: dev.NttPlan(f, prm))
p2 = trial("plan create 128 (second)", lambda: dev.NttPlan(f, prm))
prm2 = find_ntt_params(256, 1 << 12)
f2 = trial("field create 256", lambda: dev.Field(256, prm2.p))
p3 = trial("plan create 256 (first)", lambda: dev.NttPlan(f2, prm2))
p4 = trial("plan create 256 (second)", lambda: dev.NttPlan(f2, prm2))
