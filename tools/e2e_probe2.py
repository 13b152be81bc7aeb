"""e2e pipeline probe: wm_ntt_host in copy mode (PCIe floor) vs forward,
forward+inverse, over chunk sizes; 256-bit n=2^16 batch 64, pinned buffers."""
import sys, statistics
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2501_07535_b200 import kernels as K
from paper_2501_07535_b200.params import find_ntt_params
N, B = 1 << 16, 64
plan = K.get_plan(256, find_ntt_params(256, N))
hi = torch.randint(0, 1 << 59, (B * N, 4), dtype=torch.int64).pin_memory()
ho = torch.empty_like(hi).pin_memory()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for chunk in (1, 2, 4, 8, 16):
    row = {"chunk": chunk}
    for mode in ("copy", "forward", "forward_inverse"):
        ms = t(lambda: plan.host_transform(hi, ho, mode=mode, word_bits=64, ref_words=4, chunk=chunk))
        row[mode] = round(ms, 3)
    print(row, flush=True)
