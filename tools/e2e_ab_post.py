"""Interleaved A/B of the host pipeline's D2H placement (WM_HOST_POST=0/1,
read per call) on the bench's in-place pinned buffer, with the two-stream
copy floor measured between them (the PCIe rate of these VMs drifts by
+-10 % between runs, so only interleaved numbers compare)."""
import json, os, statistics, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2501_07535_b200 import kernels as K
from paper_2501_07535_b200.params import find_ntt_params
N, B = 1 << 16, 64
plan = K.get_plan(256, find_ntt_params(256, N))
h = torch.randint(0, 1 << 59, (B * N, 4), dtype=torch.int64).pin_memory()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
dev_buf = torch.empty(h.shape, dtype=h.dtype, device="cuda"); dev_src = torch.empty_like(dev_buf)
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream(); st = torch.cuda.current_stream()
def copies():
    s_in.wait_stream(st); s_out.wait_stream(st)
    with torch.cuda.stream(s_in): dev_buf.copy_(h, non_blocking=True)
    with torch.cuda.stream(s_out): h.copy_(dev_src, non_blocking=True)
    st.wait_stream(s_in); st.wait_stream(s_out)
settings = [("post0", {"WM_HOST_POST": "0"}), ("post1", {"WM_HOST_POST": "1"}),
            ("post1_ramp1", {"WM_HOST_POST": "1", "WM_HOST_RAMP": "1"}),
            ("post1_ramp2", {"WM_HOST_POST": "1", "WM_HOST_RAMP": "2"})]
rows = {k: [] for k in ["floor"] + [name for name, _ in settings]}
for rep in range(6):
    rows["floor"].append(t(copies))
    for name, env in settings:
        for k in ("WM_HOST_POST", "WM_HOST_RAMP"):
            os.environ.pop(k, None)
        os.environ.update(env)
        rows[name].append(t(lambda: plan.host_transform(h, h, mode="forward_inverse", word_bits=64, ref_words=4,
                                                          chunk=0)))
print(json.dumps({k: {"median_ms": round(statistics.median(v), 3), "all": [round(x, 3) for x in v]} for k, v in rows.items()}))
