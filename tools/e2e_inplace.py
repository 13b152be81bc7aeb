"""e2e host pipeline: separate in/out pinned buffers vs one buffer in place."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2501_07535_b200 import kernels as K
from paper_2501_07535_b200.params import find_ntt_params
N, B = 1 << 16, 64
plan = K.get_plan(256, find_ntt_params(256, N))
mode = sys.argv[1]
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3 / 128
a = torch.randint(0, 1 << 59, (B * N, 4), dtype=torch.int64).pin_memory()
b = a if mode == "inplace" else torch.empty_like(a).pin_memory()
ref = a.clone()
print(mode, [round(t(lambda: plan.host_transform(a, b, mode="forward_inverse", word_bits=64, ref_words=4)), 2) for _ in range(3)],
      torch.equal(b, ref), flush=True)
if len(sys.argv) > 2:
    import subprocess, time
    F = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    p = subprocess.Popen(["nvidia-smi", f"--query-gpu={F}", "--format=csv,noheader,nounits", "-lms", "100", "-i", "0"],
                         stdout=subprocess.DEVNULL)
    time.sleep(2.0)
    print("during nvidia-smi", [round(t(lambda: plan.host_transform(a, b, mode="forward_inverse", word_bits=64, ref_words=4)), 2) for _ in range(2)], flush=True)
    p.terminate(); p.wait()
    print("after nvidia-smi", [round(t(lambda: plan.host_transform(a, b, mode="forward_inverse", word_bits=64, ref_words=4)), 2) for _ in range(3)], flush=True)
