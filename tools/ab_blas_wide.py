"""A/B of vmul/axpy at wide limb counts (512/768/1024 bits, n = 2^22..2^24)
for library variants (WM_LIB_PATH per child process), both reductions and
both product strategies; GB/s of algorithmic traffic (3 x 4K bytes/element).

    python tools/ab_blas_wide.py paper_2501_07535_b200/libwidemod_b200.so [other.so ...]
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CHILD = r'''
import sys, json, statistics
sys.path.insert(0, %r)
import torch
from paper_2501_07535_b200 import device as dev
from paper_2501_07535_b200.params import find_ntt_params
def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)
res = {}
for bits, n in ((512, 1 << 24), (768, 1 << 24), (1024, 1 << 23)):
    Kl = bits // 32
    a = torch.randint(0, 1 << 27, (n, Kl), dtype=torch.int32, device="cuda"); b = a.flip(0).contiguous()
    o = torch.empty_like(a)
    q = find_ntt_params(bits, 1).p
    ref = None
    for red in ("auto", "barrett"):
        for strat in ("schoolbook", "karatsuba"):
            f = dev.Field(bits, q, strat, reduction=red)
            got = f.vmul(a[:4096], b[:4096])
            ref = got if ref is None else ref
            assert torch.equal(got, ref)
            mv = t(lambda: f.vmul(a, b, out=o))
            ma = t(lambda: f.axpy(12345, a, b, out=o))
            tag = f"{bits}_{f.reduction[:2]}_{strat[:4]}"
            res[f"vmul{tag}"] = round(3 * 4 * Kl * n / mv / 1e6, 1)
            res[f"axpy{tag}"] = round(3 * 4 * Kl * n / ma / 1e6, 1)
    del a, b, o
print(json.dumps(res))
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, WM_LIB_PATH=str(ROOT / lib))
    out = subprocess.run([sys.executable, "-c", CHILD % (str(ROOT),)], env=env, capture_output=True, text=True)
    print(lib, out.stdout.strip() or out.stderr[-2000:], flush=True)
