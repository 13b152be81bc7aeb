"""Measure pinned H2D / D2H bandwidth and whether the two directions overlap."""
import torch, time
n = 128 << 20
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
h2d = timeit(lambda: d_a.copy_(h_in, non_blocking=True))
d2h = timeit(lambda: h_out.copy_(d_b, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
bi = timeit(both)
print(f"H2D {n/h2d/1e9:.1f} GB/s  D2H {n/d2h/1e9:.1f} GB/s  both-concurrent {2*n/bi/1e9:.1f} GB/s aggregate ({bi*1e3:.2f} ms vs {1e3*(h2d+d2h):.2f} serial)")
print("cpu count", __import__('os').cpu_count(), torch.cuda.get_device_name())
