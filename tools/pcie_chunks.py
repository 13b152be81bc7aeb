"""Chunked bidirectional PCIe copies (the wm_ntt_host pattern without kernels):
H2D chunk c on one stream, D2H chunk c (after its H2D) on another, over
128 MiB each way; compares with single 128 MiB copies."""
import time, torch
n = 128 << 20
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(chunk):
    evs = []
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    for off in range(0, n, chunk):
        with torch.cuda.stream(s1):
            d[off:off + chunk].copy_(h_in[off:off + chunk], non_blocking=True)
            e = torch.cuda.Event(); e.record(s1)
        s2.wait_event(e)
        with torch.cuda.stream(s2):
            h_out[off:off + chunk].copy_(d[off:off + chunk], non_blocking=True)
    cur.wait_stream(s2); cur.wait_stream(s1)
for chunk in (1 << 20, 2 << 20, 4 << 20, 8 << 20, 16 << 20, 32 << 20):
    run(chunk); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): run(chunk)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"chunk {chunk >> 20:3d} MiB: {ms:.3f} ms for 128 MiB each way -> {2 * n / ms / 1e6:.1f} GB/s aggregate", flush=True)
