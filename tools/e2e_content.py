"""Bisect the bench-process e2e slowdown: set_device, device buffers allocated
before the first e2e call."""
import sys
sys.path.insert(0, '.')
import torch, bench
from paper_2501_07535_b200 import kernels as K
from paper_2501_07535_b200.params import find_ntt_params
mode = sys.argv[1]
if "setdev" in mode:
    torch.cuda.set_device(0)
N, B = 1 << 16, 64
plan = K.get_plan(256, find_ntt_params(256, N))
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3 / 128
keep = []
if "alloc" in mode:
    x = bench.canonical_random(torch, B * N, 1234)
    keep += [x, torch.empty_like(x), torch.empty_like(x),
             torch.empty(plan.workspace_bytes(B) // 4, dtype=torch.int32, device="cuda"),
             torch.empty(2 * bench.L2_BYTES // 4, dtype=torch.int32, device="cuda")]
a = bench.e2e_host_buffers(torch, plan.field)[0]
print(mode, [round(t(lambda: plan.host_transform(a, a, mode="forward_inverse", word_bits=64, ref_words=4)), 2) for _ in range(3)], flush=True)
