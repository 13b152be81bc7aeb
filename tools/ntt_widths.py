"""NTT bit-width sweep: forward+inverse n=2^16 (and 2^12) batch 64 at
64/128/256/384/512/768/1024 bits, us per transform and ns per butterfly
(the paper's per-butterfly metric)."""
import json, statistics, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2501_07535_b200 import kernels as K
from paper_2501_07535_b200.params import find_ntt_params

def t(fn, reps=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)

for logn in (12, 16):
    n, B = 1 << logn, 64
    for bits in (64, 128, 256, 384, 512, 768, 1024):
        Kl = (bits + 31) // 32
        try:
            plan = K.get_plan(bits, find_ntt_params(bits, n))
        except Exception as exc:
            print(json.dumps({"bits": bits, "logn": logn, "error": str(exc)[:120]})); continue
        x = torch.randint(0, 1 << 30, (B * n, Kl), dtype=torch.int32, device="cuda")
        x[:, Kl - 1] &= (1 << (bits - 5 - 32 * (Kl - 1))) - 1
        y = torch.empty_like(x); z = torch.empty_like(x)
        ws = torch.empty(max(1, plan.workspace_bytes(B) // 4), dtype=torch.int32, device="cuda")
        ms = t(lambda: (plan.forward(x, out=y, workspace=ws), plan.inverse(y, out=z, workspace=ws)))
        assert torch.equal(z, x)
        us = ms * 1e3 / (2 * B)
        print(json.dumps({"bits": bits, "logn": logn, "passes": plan.pass_log_sizes, "us_per_transform": round(us, 3),
                          "ns_per_butterfly": round(us * 1e3 / (n // 2 * logn), 4)}), flush=True)
        del x, y, z, ws
