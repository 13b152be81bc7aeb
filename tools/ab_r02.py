"""A/B timing of library variants (round 2): the headline NTT (256-bit
n=2^16 batch 64 fwd+inv) with the auto-selected reduction and with
reduction="barrett", and vmul/axpy at n=2^24 for 128/256/384/768 bits with
both reductions and both product strategies.  Each variant runs in its own
process (WM_LIB_PATH selects the .so).

    python tools/ab_r02.py paper_2501_07535_b200/libwidemod_b200.so [other.so ...]
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
N, B = 1 << 16, 64
prm = find_ntt_params(256, N)
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        flush.add_(1)
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)
res = {}
x = torch.randint(0, 1 << 27, (B * N, 8), dtype=torch.int32, device="cuda")
y = torch.empty_like(x); z = torch.empty_like(x)
for red in ("auto", "barrett"):
    f = dev.Field(256, prm.p, reduction=red)
    plan = dev.NttPlan(f, prm)
    ws = torch.empty(max(1, plan.workspace_bytes(B) // 4), dtype=torch.int32, device="cuda")
    ms = t(lambda: (plan.forward(x, out=y, workspace=ws), plan.inverse(y, out=z, workspace=ws)))
    assert torch.equal(z, x)
    p0 = t(lambda: plan.run_pass(0, x, y))
    p1 = t(lambda: plan.run_pass(1, x, y))
    res[f"ntt_{f.reduction}"] = {"us_per_transform": round(ms * 1e3 / 128, 3), "pass0_us": round(p0 * 1e3, 1),
                                 "pass1_us": round(p1 * 1e3, 1)}
    del plan, ws
del x, y, z
n = 1 << 24
for bits in %r:
    Kl = bits // 32
    a = torch.randint(0, 1 << 27, (n, Kl), dtype=torch.int32, device="cuda"); b = a.flip(0).contiguous()
    o = torch.empty_like(a)
    q = find_ntt_params(bits, 1).p
    for red in ("auto", "barrett"):
        for strat in ("schoolbook", "karatsuba"):
            f = dev.Field(bits, q, strat, reduction=red)
            mv = t(lambda: f.vmul(a, b, out=o))
            ma = t(lambda: f.axpy(12345, a, b, out=o))
            tag = f"{bits}_{f.reduction[:2]}_{strat[:4]}"
            res[f"vmul{tag}"] = round(3 * 4 * Kl * n / mv / 1e6, 1)
            res[f"axpy{tag}"] = round(3 * 4 * Kl * n / ma / 1e6, 1)
    del a, b, o
print(json.dumps(res))
'''
bits = [128, 256, 384, 768]
for lib in sys.argv[1:]:
    env = dict(os.environ, WM_LIB_PATH=str(ROOT / lib))
    out = subprocess.run([sys.executable, "-c", CHILD % (str(ROOT), bits)], env=env, capture_output=True, text=True)
    print(lib, out.stdout.strip() or out.stderr[-2000:], flush=True)
