"""A/B timing of library variants on the headline NTT (256-bit, n=2^16,
batch 64, forward+inverse) and 256-bit vmul n=2^22; each variant in its own
process (WM_LIB_PATH selects the .so).  Variants are built with
_build.build(variant=..., defines=...), typically restricted to K=8 via
-D'WM_BLAS_KS(X)=X(8)' -D'WM_NTT_KS(X)=X(8)'."""
import json, os, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
CHILD = r'''
import sys, json, statistics
sys.path.insert(0, %r)
import torch
from paper_2501_07535_b200 import kernels as K, device as dev
from paper_2501_07535_b200.params import find_ntt_params
N, B = 1 << 16, 64
plan = K.get_plan(256, find_ntt_params(256, N))
x = torch.randint(0, 1 << 27, (B * N, 8), dtype=torch.int32, device="cuda")
y = torch.empty_like(x); z = torch.empty_like(x)
ws = torch.empty(plan.workspace_bytes(B) // 4, dtype=torch.int32, device="cuda")
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)
ms = t(lambda: (plan.forward(x, out=y, workspace=ws), plan.inverse(y, out=z, workspace=ws)))
assert torch.equal(z, x)
p0 = t(lambda: plan.run_pass(0, x, y)); p1 = t(lambda: plan.run_pass(1, x, y))
res = {"us_per_transform": round(ms * 1e3 / 128, 3), "pass0_us": round(p0 * 1e3, 1), "pass1_us": round(p1 * 1e3, 1)}
n = 1 << 22
a = torch.randint(0, 1 << 27, (n, 8), dtype=torch.int32, device="cuda"); b = a.flip(0).contiguous()
o = torch.empty_like(a)
f = dev.Field(256, find_ntt_params(256, 1).p)
res["vmul256_GBps"] = round(96 * n / t(lambda: f.vmul(a, b, out=o)) / 1e6, 1)
fk = dev.Field(256, find_ntt_params(256, 1).p, "karatsuba")
res["vmul256_kara_GBps"] = round(96 * n / t(lambda: fk.vmul(a, b, out=o)) / 1e6, 1)
ref = f.vmul(a, b, out=torch.empty_like(a)); assert torch.equal(fk.vmul(a, b, out=o), ref)
print(json.dumps(res))
''' % str(ROOT)
for lib in sys.argv[1:]:
    env = dict(os.environ, WM_LIB_PATH=str(ROOT / lib))
    out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(Path(lib).name, out.stdout.strip() or out.stderr[-2000:], flush=True)
