"""A/B of the light BLAS kernels (vadd at 128/256 bits, vmul/axpy at 128)
against the reference's emitted CUDA kernels (oracle/_ref/libref_gpu.so) in
the same process, for each library variant given (WM_LIB_PATH per child).

    python tools/ab_light_blas.py paper_2501_07535_b200/libwidemod_b200.so [variant.so ...]
"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CHILD = r'''
import sys, json, ctypes, statistics
sys.path.insert(0, %r)
import torch
from paper_2501_07535_b200 import device as dev
from paper_2501_07535_b200 import kernels as K
from paper_2501_07535_b200.params import find_ntt_params, compute_barrett
lib = ctypes.CDLL(%r + "/oracle/_ref/libref_gpu.so")
vp, i = ctypes.c_void_p, ctypes.c_int
def timed(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)
n = 1 << 24
res = {}
for bits in (128, 256):
    Kl = bits // 32
    q = find_ntt_params(bits, 1).p
    f = dev.Field(bits, q)
    a = torch.randint(0, 1 << 27, (n, Kl), dtype=torch.int32, device="cuda")
    b = a.flip(0).contiguous()
    o = torch.empty_like(a)
    ra, rb = f.to_ref_layout(a, 32, Kl), f.to_ref_layout(b, 32, Kl)
    ro = torch.empty_like(ra)
    gb = 3 * 4 * Kl * n / 1e9
    words = lambda v: torch.tensor([w - (1 << 32) if w >= 1 << 31 else w for w in K.to_words(v, Kl, 32)], dtype=torch.int32).cuda()
    for kind in ("vadd", "vmul", "axpy"):
        if bits == 256 and kind != "vadd":
            continue
        ours = (lambda: f.axpy(12345, a, b, out=o)) if kind == "axpy" else (lambda kind=kind: getattr(f, kind)(a, b, out=o))
        res[f"{kind}{bits}_ours"] = round(gb / timed(ours) * 1e3, 1)
        fn = getattr(lib, f"refdrv_{kind}{n}_{bits}w32_baked")
        args = ([words(12345), ra] if kind == "axpy" else [ra, rb]) + ([rb] if kind == "axpy" else [])
        fn.argtypes = [vp] * (len(args) + 1) + [i, i]
        ptrs = [t.data_ptr() for t in args]
        res[f"{kind}{bits}_ref_baked"] = round(gb / timed(lambda: fn(*ptrs, ro.data_ptr(), n, 256)) * 1e3, 1)
    del a, b, o, ra, rb, ro
# copy roofline in the same process
src = torch.empty(1 << 29, dtype=torch.int32, device="cuda"); dst = torch.empty_like(src)
res["copy_GBps"] = round(2 * 4 * src.numel() / 1e9 / timed(lambda: dst.copy_(src)) * 1e3, 1)
print(json.dumps(res))
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, WM_LIB_PATH=str(ROOT / lib))
    for rep in range(2):
        out = subprocess.run([sys.executable, "-c", CHILD % (str(ROOT), str(ROOT))], env=env, capture_output=True,
                             text=True)
        print(lib, out.stdout.strip() or out.stderr[-2000:], flush=True)
