"""Chunked copy timeline (round 2 e2e diagnosis): H2D chunk c on one
stream, D2H of chunk c on another after it, with timing events, on the
bench's in-place pinned buffer; prints per-chunk start/end (ms) and the
total against the whole-buffer two-stream floor."""
import json, sys
import torch
N, B = 1 << 16, 64
h = torch.randint(0, 1 << 59, (B * N, 4), dtype=torch.int64).pin_memory()
flat = h.view(-1)
d = torch.empty(flat.numel(), dtype=torch.int64, device="cuda")
s_in, s_out, st = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.current_stream()
def run(chunk_elems, lead, record=False):
    n = flat.numel()
    cs = list(range(0, n, chunk_elems))
    ev_in = [torch.cuda.Event(enable_timing=record) for _ in cs]
    ev_out = [torch.cuda.Event(enable_timing=record) for _ in cs]
    ev_s = [torch.cuda.Event(enable_timing=record) for _ in cs]
    ev_so = [torch.cuda.Event(enable_timing=record) for _ in cs]
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record(st)
    s_in.wait_stream(st); s_out.wait_stream(st)
    for i, c0 in enumerate(cs):
        c1 = min(n, c0 + chunk_elems)
        with torch.cuda.stream(s_in):
            if i >= lead: s_in.wait_event(ev_out[i - lead])
            if record: ev_s[i].record(s_in)
            d[c0:c1].copy_(flat[c0:c1], non_blocking=True)
            ev_in[i].record(s_in)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_in[i])
            if record: ev_so[i].record(s_out)
            flat[c0:c1].copy_(d[c0:c1], non_blocking=True)
            ev_out[i].record(s_out)
    st.wait_stream(s_out)
    t1.record(st)
    torch.cuda.synchronize()
    total = t0.elapsed_time(t1)
    tl = None
    if record:
        tl = [(round(t0.elapsed_time(ev_s[i]), 3), round(t0.elapsed_time(ev_in[i]), 3),
               round(t0.elapsed_time(ev_so[i]), 3), round(t0.elapsed_time(ev_out[i]), 3)) for i in range(len(cs))]
    return total, tl
res = {}
for mib in (2, 8, 32):
    ce = mib * (1 << 20) // 8
    for lead in (1, 2, 4, 64):
        run(ce, lead)
        res[f"{mib}MiB_lead{lead}"] = round(min(run(ce, lead)[0] for _ in range(3)), 3)
tot, tl = run(8 * (1 << 20) // 8, 64, record=True)
def floor():
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    d2 = torch.empty_like(d)
    t0.record(st); s_in.wait_stream(st); s_out.wait_stream(st)
    with torch.cuda.stream(s_in): d.copy_(flat, non_blocking=True)
    with torch.cuda.stream(s_out): flat.copy_(d2, non_blocking=True)
    st.wait_stream(s_in); st.wait_stream(s_out); t1.record(st); torch.cuda.synchronize()
    return t0.elapsed_time(t1)
floor(); res["floor"] = round(min(floor() for _ in range(3)), 3)
h2 = torch.randint(0, 1 << 59, (B * N, 4), dtype=torch.int64).pin_memory()
def floor_sep():
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    d2 = torch.empty_like(d)
    t0.record(st); s_in.wait_stream(st); s_out.wait_stream(st)
    with torch.cuda.stream(s_in): d.copy_(flat, non_blocking=True)
    with torch.cuda.stream(s_out): h2.view(-1).copy_(d2, non_blocking=True)
    st.wait_stream(s_in); st.wait_stream(s_out); t1.record(st); torch.cuda.synchronize()
    return t0.elapsed_time(t1)
floor_sep(); res["floor_two_buffers"] = round(min(floor_sep() for _ in range(3)), 3)
def h2d_only():
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record(st); d.copy_(flat, non_blocking=True); t1.record(st); torch.cuda.synchronize()
    return t0.elapsed_time(t1)
def d2h_only():
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record(st); flat.copy_(d, non_blocking=True); t1.record(st); torch.cuda.synchronize()
    return t0.elapsed_time(t1)
h2d_only(); d2h_only()
res["h2d_only"] = round(min(h2d_only() for _ in range(3)), 3)
res["d2h_only"] = round(min(d2h_only() for _ in range(3)), 3)
print(json.dumps(res))
print(json.dumps({"timeline_8MiB_lead64 (h2d start, h2d end, d2h start, d2h end)": tl[:6] + ["..."] + tl[-4:]}))
