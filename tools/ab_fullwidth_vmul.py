"""A/B of library variants on full-width (Montgomery-field) vmul at 256/384/768 bits."""
import json, os, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
CHILD = r'''
import sys, json, statistics
sys.path.insert(0, %r)
import torch
from paper_2501_07535_b200 import device as dev
def t(fn, reps=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)
Q = {256: 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001,
     384: int("1a0111ea397fe69a4b1ba7b6434bacd764774b84f38512bf6730d2a0f6b0f6241eabfffeb153ffffb9feffffffffaaab", 16),
     768: 2**768 - 1}
res = {}
for bits, q in Q.items():
    Kl = bits // 32; n = 1 << 24
    a = torch.randint(0, 1 << 27, (n, Kl), dtype=torch.int32, device="cuda"); b = a.flip(0).contiguous(); o = torch.empty_like(a)
    f = dev.Field(bits, q, "montgomery")
    res[f"vmul{bits}"] = round(12 * Kl * n / t(lambda: f.vmul(a, b, out=o)) / 1e6, 1)
    del a, b, o
print(json.dumps(res))
''' % str(ROOT)
for lib in sys.argv[1:]:
    env = dict(os.environ, WM_LIB_PATH=str(ROOT / lib))
    out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(Path(lib).name, out.stdout.strip() or out.stderr[-1500:], flush=True)
