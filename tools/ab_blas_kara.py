"""A/B: vadd/vmul/axpy at 128/256/384/768 bits with the bench's strategies."""
import json, os, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
CHILD = r'''
import sys, json, statistics
sys.path.insert(0, %r)
import torch
from paper_2501_07535_b200 import device as dev
from paper_2501_07535_b200.params import find_ntt_params
def t(fn, reps=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)
res = {}
for bits in (128, 256, 384, 768):
    Kl = bits // 32; n = 1 << 24
    a = torch.randint(0, 1 << 27, (n, Kl), dtype=torch.int32, device="cuda"); b = a.flip(0).contiguous(); o = torch.empty_like(a)
    q = find_ntt_params(bits, 1).p
    for strat in ("schoolbook", "karatsuba"):
        f = dev.Field(bits, q, strat)
        res[f"vmul{bits}_{strat[:4]}"] = round(12 * Kl * n / t(lambda: f.vmul(a, b, out=o)) / 1e6, 1)
        res[f"axpy{bits}_{strat[:4]}"] = round(12 * Kl * n / t(lambda: f.axpy(12345, a, b, out=o)) / 1e6, 1)
    del a, b, o
print(json.dumps(res))
''' % str(ROOT)
for lib in sys.argv[1:]:
    env = dict(os.environ, WM_LIB_PATH=str(ROOT / lib))
    out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(Path(lib).name, out.stdout.strip() or out.stderr[-1500:], flush=True)
