import sys, json, statistics, os
sys.path.insert(0, '.')
import torch
from paper_2501_07535_b200 import device as dev
from paper_2501_07535_b200.params import NttParams
sys.path.insert(0, 'tests')
def t(fn, reps=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)
from test_fullwidth_gpu import _prime, _params
res = {}
for bits in (256, 512, 768, 1024):
    p = _prime("random", bits) if bits != 256 else 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001
    n, B = 1 << 16, 64
    f = dev.Field(bits, p, "montgomery"); plan = dev.NttPlan(f, _params(p, n)); K = f.limbs
    x = torch.randint(0, 1 << 30, (B * n, K), dtype=torch.int32, device="cuda"); x[:, K - 1] &= (1 << 29) - 1
    y = torch.empty_like(x); z = torch.empty_like(x)
    ws = torch.empty(max(1, plan.workspace_bytes(B) // 4), dtype=torch.int32, device="cuda")
    ms = t(lambda: (plan.forward(x, out=y, workspace=ws), plan.inverse(y, out=z, workspace=ws)))
    assert torch.equal(z, x)
    res[f"mont{bits}"] = round(ms * 1e3 / 128, 2)
    del x, y, z, ws
print(os.environ.get("WM_LIB_PATH"), json.dumps(res))
