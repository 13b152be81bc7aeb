"""Break down the end-to-end host-buffer path: copies, layout kernels, NTTs."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2501_07535_b200 import kernels as K
from paper_2501_07535_b200.params import find_ntt_params
N, B = 1 << 16, 64
plan = K.get_plan(256, find_ntt_params(256, N))
f = plan.field
x = torch.randint(0, 1 << 27, (B * N, 8), dtype=torch.int32, device="cuda")
ref = f.to_ref_layout(x, 64, 4)
h_in = torch.empty(ref.shape, dtype=torch.int64, pin_memory=True); h_in.copy_(ref.cpu())
h_out = torch.empty(h_in.shape, dtype=h_in.dtype, pin_memory=True)
y = torch.empty_like(x); z = torch.empty_like(x)
ws = torch.empty(plan.workspace_bytes(B) // 4, dtype=torch.int32, device="cuda")
def t(name, fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    print(f"{name:28s} {e0.elapsed_time(e1)/reps:8.3f} ms")
t("h2d 128MiB", lambda: ref.copy_(h_in, non_blocking=True))
t("d2h 128MiB", lambda: h_out.copy_(ref, non_blocking=True))
t("ref_to_limbs", lambda: f.from_ref_layout(ref, 64, 4, out=y))
t("limbs_to_ref", lambda: f.to_ref_layout(y, 64, 4, out=ref))
t("fwd+inv", lambda: (plan.forward(x, out=y, workspace=ws), plan.inverse(y, out=z, workspace=ws)))
for chunk in (0, 2, 4, 8, 16, 32):
    t(f"host_transform chunk={chunk}", lambda: plan.host_transform(h_in, h_out, "forward_inverse", 64, 4, chunk))
