"""e2e pipeline probe (round 2): wm_ntt_host on the bench's single in-place
pinned buffer, copy mode vs forward+inverse over chunk sizes (0 = auto), and
the two-stream whole-buffer copy floor; 256-bit n=2^16 batch 64."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2501_07535_b200 import kernels as K
from paper_2501_07535_b200.params import find_ntt_params
N, B = 1 << 16, 64
plan = K.get_plan(256, find_ntt_params(256, N))
h = torch.randint(0, 1 << 59, (B * N, 4), dtype=torch.int64).pin_memory()
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
dev_buf = torch.empty(h.shape, dtype=h.dtype, device="cuda"); dev_src = torch.empty_like(dev_buf)
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
st = torch.cuda.current_stream()
def copies():
    s_in.wait_stream(st); s_out.wait_stream(st)
    with torch.cuda.stream(s_in): dev_buf.copy_(h, non_blocking=True)
    with torch.cuda.stream(s_out): h.copy_(dev_src, non_blocking=True)
    st.wait_stream(s_in); st.wait_stream(s_out)
res = {"floor_ms": round(t(copies), 3)}
for chunk in (0, 1, 2, 4, 8, 16):
    for mode in ("copy", "forward_inverse"):
        res[f"{mode}_c{chunk}"] = round(t(lambda: plan.host_transform(h, h, mode=mode, word_bits=64, ref_words=4,
                                                                      chunk=chunk)), 3)
res["floor_ms_again"] = round(t(copies), 3)
print(json.dumps(res))
