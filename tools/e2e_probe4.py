"""e2e pipeline A/B (round 2): H2D lead over D2H (WM_HOST_AHEAD, read once
per process) x chunk size, copy mode and forward+inverse, against the
two-stream whole-buffer copy floor; each setting in its own process."""
import json, os, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
CHILD = r'''
import json, sys
sys.path.insert(0, %r)
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
res = {}
for chunk in (0, 4, 8, 16):
    for mode in ("copy", "forward_inverse"):
        res[f"{mode}_c{chunk}"] = round(t(lambda: plan.host_transform(h, h, mode=mode, word_bits=64, ref_words=4, chunk=chunk)), 3)
dev_buf = torch.empty(h.shape, dtype=h.dtype, device="cuda"); dev_src = torch.empty_like(dev_buf)
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream(); st = torch.cuda.current_stream()
def copies():
    s_in.wait_stream(st); s_out.wait_stream(st)
    with torch.cuda.stream(s_in): dev_buf.copy_(h, non_blocking=True)
    with torch.cuda.stream(s_out): h.copy_(dev_src, non_blocking=True)
    st.wait_stream(s_in); st.wait_stream(s_out)
res["floor"] = round(t(copies), 3)
print(json.dumps(res))
'''
settings = [(a, p) for p in (0, 1) for a in (2, 3, 4, 8)] if len(sys.argv) < 2 else \
    [tuple(int(v) for v in x.split(",")) for x in sys.argv[1:]]
for ahead, post in settings:
    env = dict(os.environ, WM_HOST_AHEAD=str(ahead), WM_HOST_POST=str(post))
    out = subprocess.run([sys.executable, "-c", CHILD % str(ROOT)], env=env, capture_output=True, text=True)
    print("ahead", ahead, "post", post, out.stdout.strip() or out.stderr[-1500:], flush=True)
