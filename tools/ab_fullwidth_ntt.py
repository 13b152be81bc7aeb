"""A/B of the full-width NTT modes (BLS12-381 r: Montgomery, MODE 1; BN254 r:
Shoup [0,4p), MODE 2) at 256 bits, n = 2^16, batch 64, forward + inverse,
for each library variant given (WM_LIB_PATH per child process)."""
import os, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
CHILD = r'''
import sys, json, statistics
sys.path.insert(0, %r)
import torch
from paper_2501_07535_b200 import device as dev
from paper_2501_07535_b200.params import NttParams
N, B = 1 << 16, 64
def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)
res = {}
for name, p, g in (("bls12_381_r", 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001, 7),
                   ("bn254_r", 21888242871839275222246405745257275088548364400416034343698204186575808495617, 5)):
    w = pow(g, (p - 1) // N, p)
    f = dev.Field(256, p, "montgomery")
    plan = dev.NttPlan(f, NttParams(n=N, p=p, root=w, root_inv=pow(w, -1, p), n_inv=pow(N, -1, p)))
    x = torch.randint(0, 1 << 28, (B * N, 8), dtype=torch.int32, device="cuda")
    y = torch.empty_like(x); z = torch.empty_like(x)
    ws = torch.empty(max(1, plan.workspace_bytes(B) // 4), dtype=torch.int32, device="cuda")
    ms = t(lambda: (plan.forward(x, out=y, workspace=ws), plan.inverse(y, out=z, workspace=ws)))
    assert torch.equal(z, x)
    res[name] = round(ms * 1e3 / (2 * B), 3)
print(json.dumps(res))
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, WM_LIB_PATH=str(ROOT / lib))
    out = subprocess.run([sys.executable, "-c", CHILD % str(ROOT)], env=env, capture_output=True, text=True)
    print(lib, out.stdout.strip() or out.stderr[-2000:], flush=True)
