"""Bisect: e2e host pipeline timing standalone vs after device-resident work
(the order bench.py uses)."""
import sys, statistics
sys.path.insert(0, '.')
import torch
from paper_2501_07535_b200 import kernels as K
from paper_2501_07535_b200.params import find_ntt_params
N, B = 1 << 16, 64
plan = K.get_plan(256, find_ntt_params(256, N))
hi = torch.randint(0, 1 << 59, (B * N, 4), dtype=torch.int64).pin_memory()
ho = torch.empty_like(hi).pin_memory()
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
e2e = lambda: plan.host_transform(hi, ho, mode="forward_inverse", word_bits=64, ref_words=4, chunk=0)
print("fresh", round(t(e2e) * 1e3 / 128, 2), flush=True)
x = torch.randint(0, 1 << 27, (B * N, 8), dtype=torch.int32, device="cuda")
y = torch.empty_like(x); z = torch.empty_like(x)
ws = torch.empty(plan.workspace_bytes(B) // 4, dtype=torch.int32, device="cuda")
flush = torch.empty(2 * 126 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
for _ in range(20):
    flush.add_(1); plan.forward(x, out=y, workspace=ws); plan.inverse(y, out=z, workspace=ws)
torch.cuda.synchronize()
print("after device work", round(t(e2e) * 1e3 / 128, 2), flush=True)
del flush
torch.cuda.synchronize()
print("after freeing flush", round(t(e2e) * 1e3 / 128, 2), flush=True)
import subprocess, time
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "100"], stdout=subprocess.DEVNULL)
time.sleep(0.5)
print("with nvidia-smi sampling", round(t(e2e) * 1e3 / 128, 2), flush=True)
p.terminate(); p.wait()
print("after nvidia-smi", round(t(e2e) * 1e3 / 128, 2), flush=True)
