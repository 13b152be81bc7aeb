import sys, types
sys.path.insert(0, '.')
import torch, bench
from paper_2501_07535_b200 import kernels as K, device as dev
from paper_2501_07535_b200.params import find_ntt_params
N, B = bench.N, bench.BATCH
plan = K.get_plan(256, find_ntt_params(256, N))
args = types.SimpleNamespace(warmup=3, steps=10, e2e_chunk=0)
print("bench.run_e2e fresh process:", bench.run_e2e(args, torch, plan, bench.e2e_host_buffers(torch, plan.field), None, 1)["value"], flush=True)
hi = torch.randint(0, 1 << 59, (B * N, 4), dtype=torch.int64).pin_memory()
ho = torch.empty_like(hi).pin_memory()
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
print("probe buffers:", t(lambda: plan.host_transform(hi, ho, mode="forward_inverse", word_bits=64, ref_words=4)) * 1e3 / 128, flush=True)
a = torch.empty((B * N, 4), dtype=torch.int64, pin_memory=True); a.copy_(hi)
b = torch.empty((B * N, 4), dtype=torch.int64, pin_memory=True)
print("empty(pin_memory) buffers:", t(lambda: plan.host_transform(a, b, mode="forward_inverse", word_bits=64, ref_words=4)) * 1e3 / 128, flush=True)
print("bench.run_e2e again:", bench.run_e2e(args, torch, plan, bench.e2e_host_buffers(torch, plan.field), None, 1)["value"], flush=True)
