"""A/B of library variants on the NTT at one width: python tools/ab_widths.py BITS LIB..."""
import json, os, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
CHILD = r'''
import sys, json, statistics
sys.path.insert(0, %r)
import torch
from paper_2501_07535_b200 import kernels as K
from paper_2501_07535_b200.params import find_ntt_params
bits = %d
Kl = (bits + 31) // 32
res = {}
for logn in (12, 16):
    n, B = 1 << logn, 64
    plan = K.get_plan(bits, find_ntt_params(bits, n))
    x = torch.randint(0, 1 << 30, (B * n, Kl), dtype=torch.int32, device="cuda")
    x[:, Kl - 1] &= (1 << (bits - 5 - 32 * (Kl - 1))) - 1
    y = torch.empty_like(x); z = torch.empty_like(x)
    ws = torch.empty(max(1, plan.workspace_bytes(B) // 4), dtype=torch.int32, device="cuda")
    def t(fn, reps=10):
        for _ in range(2): fn()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for a, b in ev:
            a.record(); fn(); b.record()
        torch.cuda.synchronize()
        return statistics.median(a.elapsed_time(b) for a, b in ev)
    ms = t(lambda: (plan.forward(x, out=y, workspace=ws), plan.inverse(y, out=z, workspace=ws)))
    assert torch.equal(z, x)
    res[f"2^{logn}_us"] = round(ms * 1e3 / 128, 3)
print(json.dumps(res))
'''
bits = int(sys.argv[1])
for lib in sys.argv[2:]:
    env = dict(os.environ, WM_LIB_PATH=str(ROOT / lib))
    out = subprocess.run([sys.executable, "-c", CHILD % (str(ROOT), bits)], env=env, capture_output=True, text=True)
    print(Path(lib).name, bits, out.stdout.strip() or out.stderr[-1500:], flush=True)
