import json, os, subprocess, sys
ROOT = "/root/repo"
CHILD = r'''
import sys, json, statistics
sys.path.insert(0, "ROOT")
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
n, B = 1 << 16, 64
for bits in (32, 64, 96, 128, 160, 192, 224, 256):
    prm = find_ntt_params(bits, n)
    f = dev.Field(bits, prm.p, reduction="barrett")
    plan = dev.NttPlan(f, prm)
    Kl = f.limbs
    x = torch.randint(0, 1 << 30, (B * n, Kl), dtype=torch.int32, device="cuda")
    x[:, Kl - 1] &= (1 << (bits - 5 - 32 * (Kl - 1))) - 1
    y = torch.empty_like(x); z = torch.empty_like(x)
    ws = torch.empty(max(1, plan.workspace_bytes(B) // 4), dtype=torch.int32, device="cuda")
    ms = t(lambda: (plan.forward(x, out=y, workspace=ws), plan.inverse(y, out=z, workspace=ws)))
    assert torch.equal(z, x)
    res[bits] = round(ms * 1e3 / (2 * B), 3)
print(json.dumps(res))
'''.replace("ROOT", ROOT)
for lib in sys.argv[1:]:
    env = dict(os.environ, WM_LIB_PATH=os.path.join(ROOT, lib))
    out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(lib, out.stdout.strip() or out.stderr[-1500:], flush=True)
