"""Benchmark: BASELINE.json's headline on the B200.

Workload (BASELINE configs[1]): 256-bit forward + inverse NTT, n = 2^16, batch
64 per GPU (weak scaling: every rank runs its own batch of 64; batched NTTs
shard by transform with no collective).  One step = 64
forward + 64 inverse transforms = 128 transforms.  metric value = microseconds
per transform over the whole job (max-over-ranks time / all transforms).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Other BASELINE configs are parity-test cases; the 256-bit vmul n=2^24 HBM
figure is reported as an extra "blas" object.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "256-bit NTT µs/transform & BLAS modmul GB/s at 1/2/4/8 B200 vs roofline"
UNIT = "us/transform"
BITS, LOGN, BATCH = 256, 16, 64
N = 1 << LOGN
K_LIMBS = 8
WORDS64 = 4  # reference layout: 256-bit = 4 x 64-bit words, MSW first
# reference algorithmic work = 3k^2 word products per butterfly
ALG_WMUL_PER_BFLY = 3 * K_LIMBS * K_LIMBS
L2_BYTES = 126 * 1024 * 1024


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------ distributed
DIST = {"backend": None}  # "nccl" | "gloo" once a process group exists


def dist_setup(gpus: int, backend: str = "auto"):
    """One process per GPU (torchrun).  backend "gloo" is the dry run of the
    N>1 accounting where NCCL cannot run: ranks share the visible GPUs
    (device = local rank mod device count), collectives go through host
    memory.  Its timings are contended and only check the plumbing."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != gpus:
        if world == 1 and gpus > 1:
            raise SystemExit("--gpus N>1 must be launched with torchrun (one process per GPU)")
    pg = None
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        use_nccl = _cuda_ok() and backend in ("auto", "nccl")
        if use_nccl:
            # bind the rank to its GPU before NCCL initialises (barriers and
            # collectives then use the right device)
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            DIST["backend"] = "nccl"
        else:
            dist.init_process_group("gloo")
            DIST["backend"] = "gloo"
        pg = dist
    return rank, world, local, pg


def device_index(local: int) -> int:
    import torch
    return local % max(1, torch.cuda.device_count())


def _cuda_ok():
    import torch
    return torch.cuda.is_available()


def barrier(pg):
    if pg is not None:
        pg.barrier()


def max_over_ranks(pg, value: float) -> float:
    if pg is None:
        return value
    import torch
    dev = "cuda" if (_cuda_ok() and DIST["backend"] == "nccl") else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.dev)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if self.proc is None or not self.path:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[2:]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, flags in rows for i, f in enumerate(flags) if f.lower() == "active"})
        loaded = [r[0] for r in rows if r[0] > 0.5 * r[1]] or [r[0] for r in rows]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------ workload
def canonical_random(torch, count: int, seed: int):
    """Uniform canonical residues for the 256-bit prime p ~ 2^252 (< 2^251)."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randint(-(1 << 31), 1 << 31, (count, K_LIMBS), dtype=torch.int32, device="cuda", generator=g)
    x[:, K_LIMBS - 1] &= (1 << 27) - 1
    return x


def flush_l2(torch, buf):
    buf.add_(1)


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def _alg_wmul(n: int) -> float:
    """SURVEY §8(d) algorithmic work of one forward 256-bit transform:
    (n/2) log2 n butterflies x 3k^2 word products."""
    return (n // 2) * (n.bit_length() - 1) * ALG_WMUL_PER_BFLY


INT_PEAK = {}  # filled by measure_int_peak() on each rank


def measure_int_peak():
    """The integer roofline, measured in this run: 32x32->64 word products
    per second of wm_probe_imad_wide (8 independent chains per thread, full
    occupancy), best of the accumulate (mode 0) and plain (mode 1) forms."""
    from paper_2501_07535_b200 import device as dev
    r0, _ = dev.probe_imad_wide(0)
    r1, _ = dev.probe_imad_wide(1)
    INT_PEAK.update({"mad_wide_per_s": r0, "mul_wide_per_s": r1, "peak_per_s": max(r0, r1)})
    return INT_PEAK["peak_per_s"]


def int_peak_wmul_per_s(sm_mhz: float | None = None):
    """Measured word-product peak (products/s); the nominal 32/clk/SM x 148
    SMs x 1965 MHz only if the probe has not run."""
    if "peak_per_s" in INT_PEAK:
        return INT_PEAK["peak_per_s"], None
    return 32 * 148 * 1965.0 * 1e6, 1965.0


def plan_work(plan, batch: int, inverse: bool) -> float:
    """Word products all passes of one direction execute for `batch`
    transforms (wm_ntt_pass_work: executed work in the plan's arithmetic)."""
    return sum(plan.pass_work(i, batch, inverse)[1] for i in range(len(plan.pass_log_sizes)))


EXTRAS = ("generic", "blas", "four_step", "batched", "reference_gpu", "full_width", "steady", "drop_in")


def want(args, name: str) -> bool:
    return not args.skip_extras and name in args.extras


def run_gpu(args, rank, world, local, pg):
    import torch

    from paper_2501_07535_b200 import device as dev
    from paper_2501_07535_b200 import kernels as K
    from paper_2501_07535_b200.params import find_ntt_params

    torch.cuda.set_device(device_index(local))
    prm = find_ntt_params(BITS, N)
    plan = K.get_plan(BITS, prm)
    field = plan.field
    stream = torch.cuda.current_stream()

    # e2e host buffer and one e2e call before the large device buffers:
    # wm_ntt_host creates its streams and device staging slots on first use,
    # and slots allocated after ~1 GB of other device buffers made every later
    # e2e step ~10 % slower on this pool (tools/e2e_bisect.py)
    bufs = e2e_host_buffers(torch, field)
    plan.host_transform(bufs[0], bufs[1], mode="forward_inverse", word_bits=64, ref_words=WORDS64,
                        chunk=args.e2e_chunk)
    torch.cuda.synchronize()

    measure_int_peak()
    x = canonical_random(torch, BATCH * N, 1234 + rank)
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    ws = torch.empty(plan.workspace_bytes(BATCH) // 4, dtype=torch.int32, device="cuda")
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device="cuda")

    def step():
        plan.forward(x, out=y, workspace=ws)
        plan.inverse(y, out=z, workspace=ws)

    launches_per_step = 2 * len(plan.pass_log_sizes)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    assert torch.equal(z, x), "INTT(NTT(x)) != x in the benchmark workload"

    # ---- device-resident timing (value): per-step events, L2 flushed between steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    fwd_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier(pg)
    torch.cuda.synchronize()
    with ClockSampler(device_index(local)) as clocks:
        for s in range(args.steps):
            flush_l2(torch, flush)
            ev[s][0].record(stream)
            step()
            ev[s][1].record(stream)
        torch.cuda.synchronize()
        # the dominant kernel alone (pass 0 = ntt_col_pass: its forward and inverse
        # launches are ~55% of the step, profiles/r01_launch_share.json), for the roofline
        for s in range(args.steps):
            flush_l2(torch, flush)
            fwd_ev[s][0].record(stream)
            plan.run_pass(0, x, y)
            fwd_ev[s][1].record(stream)
        torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    local_total_ms = sum(step_ms)
    barrier(pg)
    total_ms = max_over_ranks(pg, local_total_ms)
    transforms = world * args.steps * 2 * BATCH
    us_per_transform = total_ms * 1e3 / transforms

    pass0_ms = statistics.mean(a.elapsed_time(b) for a, b in fwd_ev)

    # ---- end-to-end through the C ABI with host buffers (reference layout),
    # before the generic-path plan and its buffers are allocated
    e2e = run_e2e(args, torch, plan, bufs, pg, world)

    # ---- the same step through the generic Barrett/Shoup path (reduction="barrett")
    generic = None
    if want(args, "generic"):
        from paper_2501_07535_b200 import device as dev
        gplan = dev.NttPlan(dev.Field(BITS, prm.p, reduction="barrett"), prm)
        gws = torch.empty(max(1, gplan.workspace_bytes(BATCH) // 4), dtype=torch.int32, device="cuda")
        for _ in range(args.warmup):
            gplan.forward(x, out=y, workspace=gws)
            gplan.inverse(y, out=z, workspace=gws)
        torch.cuda.synchronize()
        assert torch.equal(z, x), "generic-path roundtrip mismatch"
        gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        barrier(pg)
        torch.cuda.synchronize()
        for s in range(args.steps):
            flush_l2(torch, flush)
            gev[s][0].record(stream)
            gplan.forward(x, out=y, workspace=gws)
            gplan.inverse(y, out=z, workspace=gws)
            gev[s][1].record(stream)
        torch.cuda.synchronize()
        gms = max_over_ranks(pg, sum(a.elapsed_time(b) for a, b in gev))
        generic = {"us_per_transform": gms * 1e3 / transforms, "reduction": "barrett",
                   "note": "the headline step with WM_FIELD_BARRETT: Shoup butterflies (MODE 0), same inputs, "
                           "same timing protocol"}
        del gplan, gws

    # ---- extras: BLAS sweep (configs[2]), four-step single 2^24 NTT (configs[4]), reference GPU code
    blas = run_blas(args, torch, field, rank, world, pg) if want(args, "blas") else None
    four = run_four_step(args, torch, rank, world, pg) if want(args, "four_step") else None
    b20 = run_batched_2p20(args, torch, rank, world, pg) if want(args, "batched") else None
    refgpu = run_reference_gpu(args, torch, plan) if (world == 1 and want(args, "reference_gpu")) else None
    fullw = run_full_width(args, torch) if want(args, "full_width") else None
    steady = run_steady_state(args, torch, plan) if want(args, "steady") else None
    dropin = run_drop_in(args, torch) if (rank == 0 and want(args, "drop_in")) else None

    return {
        "us_per_transform": us_per_transform,
        "ms_per_step": total_ms / args.steps,
        "pass0_ms": pass0_ms,
        "pass0_work": plan.pass_work(0, BATCH, False),
        "plan_mode": {"special_form": 3, "barrett": 0}.get(field.reduction, "?"),
        "reduction": field.reduction,
        "pass_log_sizes": plan.pass_log_sizes,
        "launches_per_step": launches_per_step,
        "clocks": clocks.summary(),
        "e2e": e2e,
        "generic": generic,
        "blas": blas,
        "four_step": four,
        "batched_2p20": b20,
        "reference_gpu": refgpu,
        "full_width": fullw,
        "steady_state": steady,
        "drop_in": dropin,
    }


def e2e_host_buffers(torch, field):
    """The step's pinned host buffer in the reference layout (AoS, 4 x 64-bit
    words MSW first per 256-bit value, kernels.to_words), transformed in place
    (wm_ntt_host reads chunk c before it writes chunk c back).  One buffer
    instead of an input and an output buffer: on the VM hosts of this pool a
    larger pinned footprint made PCIe transfers 5-30 % slower and erratic
    (tools/e2e_inplace.py, profiles/r01_e2e_ab.txt).  Allocated before the
    device-resident timing for the same reason."""
    src = canonical_random(torch, BATCH * N, 99)
    host = field.to_ref_layout(src, 64, WORDS64).cpu().pin_memory()
    return host, host


def run_e2e(args, torch, plan, bufs, pg, world):
    """Public API end to end: pinned HOST buffers in the reference layout
    through the pipelined C ABI call wm_ntt_host (chunked H2D / layout
    convert + NTT + INTT + convert / D2H on overlapping streams)."""
    host_in, host_out = bufs
    stream = torch.cuda.current_stream()

    def step():
        plan.host_transform(host_in, host_out, mode="forward_inverse", word_bits=64, ref_words=WORDS64,
                            chunk=args.e2e_chunk)

    want = host_in.clone()  # forward+inverse in place leaves the buffer unchanged; checked after timing
    for _ in range(max(1, args.warmup)):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(pg)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(pg, e0.elapsed_time(e1))
    # (no host-side tensor work between the warm-up and the timed calls: torch's
    # CPU thread pool stays busy-waiting after such work and slows the enqueue)
    assert torch.equal(host_out, want), "e2e roundtrip mismatch"
    del want
    # PCIe floor: the same bytes as one H2D and one D2H copy running
    # concurrently on two streams (no kernels, no chunking)
    dev_buf = torch.empty(host_in.shape, dtype=host_in.dtype, device="cuda")
    dev_src = torch.empty_like(dev_buf)
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

    def copies():
        s_in.wait_stream(stream)
        s_out.wait_stream(stream)
        with torch.cuda.stream(s_in):
            dev_buf.copy_(host_in, non_blocking=True)
        with torch.cuda.stream(s_out):
            host_out.copy_(dev_src, non_blocking=True)
        stream.wait_stream(s_in)
        stream.wait_stream(s_out)

    copies()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        copies()
    e1.record(stream)
    torch.cuda.synchronize()
    floor_ms = max_over_ranks(pg, e0.elapsed_time(e1))
    del dev_buf, dev_src
    nbytes = host_in.numel() * host_in.element_size()
    return {"value": ms * 1e3 / (world * args.steps * 2 * BATCH), "unit": UNIT,
            "pcie_floor": floor_ms * 1e3 / (world * args.steps * 2 * BATCH),
            "pcie_floor_basis": "the step's H2D and D2H bytes as two concurrent whole-buffer copies "
                                "(pinned host <-> device, no kernels), same unit",
            "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
            "path": "NttPlan.host_transform -> C ABI wm_ntt_host(mode=FWD_INV): pinned host buffer "
                    "(reference layout) transformed in place, chunked H2D/compute/D2H pipeline",
            "chunk_transforms": args.e2e_chunk or "auto"}


def run_blas(args, torch, _field, rank, world, pg):
    """BASELINE configs[2]: vadd/vmul/axpy n=2^24 at 128/256/384/768 bits,
    device-resident (inputs > L2), GB/s of algorithmic traffic (3 x 4K bytes
    per element) vs the measured HBM copy bandwidth.  The vector is sharded
    by rank (contiguous n/P slices, no collective): every
    rank runs its slice, the launch time is the max over ranks, GB/s is the
    whole vector's bytes over that time.  vmul/axpy run with the reduction the
    field selects (two-fold for these special-form moduli) and, beside it,
    the generic Barrett path (reduction="barrett")."""
    from paper_2501_07535_b200 import device as dev
    from paper_2501_07535_b200 import dist as D
    from paper_2501_07535_b200.params import find_ntt_params
    n = 1 << 24
    lo, hi = D.shard_range(n, rank, world)
    m = hi - lo
    hbm = peaks().get("hbm_gbs", 6650.0)
    out_rows = []
    stream = torch.cuda.current_stream()
    for bits in args.blas_bits:
        K = (bits + 31) // 32
        q = find_ntt_params(bits, 1).p
        g = torch.Generator(device="cuda").manual_seed(bits * 1000 + rank)
        a = torch.randint(-(1 << 31), 1 << 31, (m, K), dtype=torch.int32, device="cuda", generator=g)
        b = torch.randint(-(1 << 31), 1 << 31, (m, K), dtype=torch.int32, device="cuda", generator=g)
        top = (1 << (bits - 5 - 32 * (K - 1))) - 1
        a[:, K - 1] &= top
        b[:, K - 1] &= top
        out = torch.empty_like(a)
        # full-product strategy per width and reduction (profiles/r02_ab_pm.txt):
        # special form: Karatsuba from 12 limbs; Barrett: from 8 limbs
        sp = "karatsuba" if K >= 12 else "schoolbook"
        sb = "karatsuba" if K >= 8 else "schoolbook"
        fields = {"vadd": [dev.Field(bits, q)],
                  "vmul": [dev.Field(bits, q, sp), dev.Field(bits, q, sb, reduction="barrett")],
                  "axpy": [dev.Field(bits, q, sp), dev.Field(bits, q, sb, reduction="barrett")]}
        for op in ("vadd", "vmul", "axpy"):
            for fm in fields[op]:
                fn = (lambda fm=fm: fm.axpy(123456789, a, b, out=out)) if op == "axpy" else \
                    (lambda op=op, fm=fm: getattr(fm, op)(a, b, out=out))
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                       for _ in range(10)]
                barrier(pg)
                torch.cuda.synchronize()
                for e0, e1 in evs:
                    e0.record(stream)
                    fn()
                    e1.record(stream)
                torch.cuda.synchronize()
                ms = max_over_ranks(pg, statistics.median(x.elapsed_time(y) for x, y in evs))
                gbs = 3 * 4 * K * n / (ms * 1e-3) / 1e9
                row = {"op": op, "bits": bits, "n": n, "ms": round(ms, 4), "GB_per_s": round(gbs, 1),
                       "hbm_frac_of_measured": round(gbs / (world * hbm), 3), "strategy": fm.strategy,
                       "reduction": fm.reduction if op != "vadd" else None}
                # binding roofline: the slower of HBM traffic and the
                # executed word products (wm_blas_work) at the measured product peak
                wp = fm.work(op)
                if wp:
                    t_int = wp * n / (world * int_peak_wmul_per_s()[0])
                    t_hbm = 3 * 4 * K * n / (world * hbm * 1e9)
                    row.update(word_products_per_elem=wp,
                               int_frac_executed=round(t_int / (ms * 1e-3), 3),
                               binding="int" if t_int > t_hbm else "hbm",
                               binding_frac=round(max(t_int, t_hbm) / (ms * 1e-3), 3))
                out_rows.append(row)
        # parity of the benchmarked slice (both reductions, all ops) against each other
        # is in tests/test_reduction_gpu.py; here a cheap cross-check of the last one
        fa, fb = fields["vmul"]
        assert torch.equal(fa.vmul(a[:4096], b[:4096]), fb.vmul(a[:4096], b[:4096])), "reduction mismatch"
        del a, b, out
    return {"rows": out_rows, "hbm_measured_gbs": hbm, "ranks": world,
            "sharding": f"contiguous n/{world} slice per rank, no collective; ms = max over ranks",
            "note": "median of 10 launches; operands 0.8-4.8 GB (> L2); bytes = 2 reads + 1 write per element; "
                    "hbm_frac_of_measured = GB/s / (ranks x measured HBM copy bandwidth); vmul/axpy rows: "
                    "int_frac_executed = word products per element (wm_blas_work) x n / time / (ranks x measured "
                    "product peak), binding = the larger of the HBM and product times, binding_frac = that time "
                    "/ measured time"}


def run_drop_in(args, torch):
    """The reference-facing calls: run_vector and
    run_ntt on Python ints at n = 2^16, 256 bits (BASELINE configs[0], one
    transform of configs[1]) — int -> limb conversion, H2D, kernels, D2H,
    limb -> int — and wm_blas_host on pinned host buffers in the reference
    layout at n = 2^24 (end-to-end BLAS GB/s beside its PCIe floor)."""
    from paper_2501_07535_b200 import device as dev
    from paper_2501_07535_b200 import kernels as K
    from paper_2501_07535_b200.params import find_ntt_params
    res = {}
    q = find_ntt_params(BITS, 1).p
    rng = np.random.Generator(np.random.PCG64(21))
    limbs = rng.integers(0, 1 << 32, size=(2 * N, K_LIMBS), dtype=np.uint64).astype(np.uint32)
    limbs[:, -1] &= (1 << 27) - 1
    vals = dev.limbs_to_ints(limbs)
    xs, ys = vals[:N], vals[N:]
    prog = K.generate_kernel(K.make_spec("vmul", BITS, 64, size=N))

    def wall(fn, reps):
        fn()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            out = fn()
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts), out

    t, out = wall(lambda: K.run_vector(prog, xs, ys), 5)
    assert out == [a * b % q for a, b in zip(xs, ys)], "run_vector mismatch"
    t_conv, _ = wall(lambda: dev.limbs_to_ints(dev.ints_to_limbs(xs, K_LIMBS)), 5)
    res["run_vector_vmul_2p16_ms"] = round(t * 1e3, 2)
    res["int_limb_roundtrip_2p16_ms"] = round(t_conv * 1e3, 2)
    prm = find_ntt_params(BITS, N)
    pn = K.generate_kernel(K.make_spec("ntt", BITS, 64, size=N))
    pi = K.generate_kernel(K.make_spec("intt", BITS, 64, size=N))
    xs = [v % prm.p for v in xs]
    t, y = wall(lambda: K.run_ntt(pn, xs), 5)
    assert K.run_ntt(pi, y) == xs, "run_ntt roundtrip mismatch"
    res["run_ntt_2p16_ms"] = round(t * 1e3, 2)
    # host-buffer BLAS (wm_blas_host), reference layout 4 x 64-bit words
    m = 1 << 24
    f = dev.Field(BITS, q)
    a = canonical_random(torch, m, 61)
    b = canonical_random(torch, m, 62)
    ah = f.to_ref_layout(a, 64, 4).cpu().pin_memory()
    bh = f.to_ref_layout(b, 64, 4).cpu().pin_memory()
    oh = torch.empty_like(ah).pin_memory()
    stream = torch.cuda.current_stream()
    for kind in ("vmul", "axpy"):
        call = (lambda: f.host_op("axpy", ah, bh, oh, scalar=12345)) if kind == "axpy" else \
            (lambda: f.host_op("vmul", ah, bh, oh))
        call()
        torch.cuda.synchronize()
        want = (f.axpy(12345, a, b) if kind == "axpy" else f.vmul(a, b))
        assert torch.equal(f.from_ref_layout(oh.cuda(), 64, 4), want), f"host {kind} mismatch"
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            call()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        res[f"host_{kind}_2p24"] = {"ms": round(ms, 3), "GB_per_s": round(3 * 32 * m / (ms * 1e-3) / 1e9, 1),
                                    "h2d_bytes": 2 * 32 * m, "d2h_bytes": 32 * m}
    # PCIe floor: the same bytes as plain copies (two H2D, one D2H, concurrent)
    da, db, do = torch.empty_like(ah, device="cuda"), torch.empty_like(bh, device="cuda"), torch.empty_like(ah, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def copies():
        s1.wait_stream(stream)
        s2.wait_stream(stream)
        with torch.cuda.stream(s1):
            da.copy_(ah, non_blocking=True)
            db.copy_(bh, non_blocking=True)
        with torch.cuda.stream(s2):
            oh.copy_(do, non_blocking=True)
        stream.wait_stream(s1)
        stream.wait_stream(s2)

    copies()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(5):
        copies()
    e1.record(stream)
    torch.cuda.synchronize()
    floor = e0.elapsed_time(e1) / 5
    res["host_blas_pcie_floor_ms"] = round(floor, 3)
    res["note"] = ("run_* medians of 5 wall-clock calls on Python ints (results checked); host_* through "
                   "Field.host_op -> wm_blas_host, pinned buffers, results checked; GB/s = 3 x 32 B x n / time")
    del a, b, ah, bh, oh, da, db, do
    torch.cuda.empty_cache()
    return res


def run_four_step(args, torch, rank, world, pg):
    """BASELINE configs[4]: one 256-bit n=2^24 NTT split four-step over all
    ranks with one NCCL all-to-all (at world=1: the same pipeline, no exchange)."""
    from paper_2501_07535_b200 import dist as D
    from paper_2501_07535_b200.params import find_ntt_params
    n = 1 << 24
    prm = find_ntt_params(BITS, n)
    if pg is None:
        comm = _SelfComm()
    elif DIST["backend"] == "gloo":
        comm = D.StagedComm()
    else:
        comm = D.TorchComm()
    torch.cuda.empty_cache()  # the BLAS sweep's multi-GB operands leave the allocator fragmented
    eng = D.FourStepNtt(BITS, prm, rank, world, comm=comm)
    L = eng.layout
    rows = L.n1 // world
    x = canonical_random(torch, rows * L.n2, 4242 + rank).view(rows, L.n2, K_LIMBS)
    for _ in range(2):
        y = eng.forward(x)
    torch.cuda.synchronize()
    back = eng.inverse(y)
    torch.cuda.synchronize()
    assert torch.equal(back, x), "four-step roundtrip mismatch"
    for _ in range(2):  # the forward's buffers cached again after the inverse's shapes
        eng.forward(x)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    reps = 5
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(pg)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps):
        eng.forward(x)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(pg, e0.elapsed_time(e1) / reps)
    a2a_bytes = (world - 1) * (n // world) * 4 * K_LIMBS // world
    res = {"n": n, "ranks": world, "ms_per_forward": round(ms, 4), "us_per_transform": round(ms * 1e3, 2),
           "split": [L.n1, L.n2], "a2a_bytes_sent_per_rank": a2a_bytes,
           "exchange": ("local copy (one rank)" if pg is None else
                        "NCCL all_to_all_single" if DIST["backend"] == "nccl" else
                        "host-staged gloo all_to_all_single (dry run: ranks share one GPU)"),
           "note": "max over ranks; forward only; input rows j1 per rank (scatter not timed)"}
    if DIST["backend"] == "gloo":
        res["fused"] = {"skipped": "symmetric-memory exchange needs one GPU per rank (gloo dry run)"}
    else:
        res["fused"] = run_four_step_fused(torch, prm, rank, world, pg, x, y, reps)
    del eng, x, y, back
    if world == 1:
        # the same transform through the single-GPU multi-pass plan (natural order in/out)
        from paper_2501_07535_b200 import kernels as K
        plan = K.get_plan(BITS, prm)
        xs = canonical_random(torch, n, 4343)
        ys = torch.empty_like(xs)
        ws = torch.empty(max(1, plan.workspace_bytes(1) // 4), dtype=torch.int32, device="cuda")
        for _ in range(2):
            plan.forward(xs, out=ys, workspace=ws)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            plan.forward(xs, out=ys, workspace=ws)
        e1.record(stream)
        torch.cuda.synchronize()
        res["single_gpu_plan_ms_per_forward"] = round(e0.elapsed_time(e1) / reps, 4)
        t = e0.elapsed_time(e1) / reps * 1e-3
        res["single_gpu_plan_int_frac_executed"] = round(plan_work(plan, 1, False) / t / int_peak_wmul_per_s()[0], 3)
        res["single_gpu_plan_int_frac_reference_work"] = round(_alg_wmul(n) / t / int_peak_wmul_per_s()[0], 3)
        res["single_gpu_plan_passes"] = plan.pass_log_sizes
        del xs, ys, ws
    torch.cuda.empty_cache()
    return res


def run_four_step_fused(torch, prm, rank, world, pg, x, y_ref, reps):
    """The same four-step with the all-to-all fused into the twiddle/transpose
    kernel: peer stores into symmetric-memory receive buffers over NVLink
    (dist.SymmComm).  At one rank a one-rank NCCL group is created for it."""
    import torch.distributed as dist
    from paper_2501_07535_b200 import dist as D
    own_group = False
    try:
        if pg is None:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ["MASTER_PORT"] = str(29500 + (os.getpid() % 2000))
            dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
            own_group = True
        n = prm.n
        comm = D.SymmComm(n // world * K_LIMBS)
        err = None
        try:
            eng = D.FourStepNtt(BITS, prm, rank, world, comm=comm)
            y = eng.forward(x)
            torch.cuda.synchronize()
            ok = bool(torch.equal(y, y_ref)) and bool(torch.equal(eng.inverse(y), x))
        except Exception as exc:  # noqa: BLE001 - agreed on below
            err = exc
        # every rank learns whether any rank failed before the timing collectives
        if pg is not None:  # pg is the torch.distributed module (dist_setup)
            flag = torch.tensor([0 if err is None else 1], dtype=torch.int32, device="cuda")
            pg.all_reduce(flag, op=pg.ReduceOp.MAX)
            if int(flag.item()) and err is None:
                err = RuntimeError("fused four-step failed on another rank")
        if err is not None:
            raise err
        stream = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier(pg)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            eng.forward(x)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = max_over_ranks(pg, e0.elapsed_time(e1) / reps)
        out = {"ms_per_forward": round(ms, 4), "matches_nccl_path": ok,
               "exchange": "wm_scale_transpose_scatter: peer stores into symmetric-memory receive buffers, "
                           "device barriers before/after"}
        del eng, comm
        return out
    except Exception as exc:  # report, keep the NCCL figure
        return {"unavailable": f"{type(exc).__name__}: {exc}"[:300]}
    finally:
        if own_group:
            dist.destroy_process_group()


def run_full_width(args, torch):
    """Full-width field (WM_FIELD_MONTGOMERY, the paper's Montgomery mode,
    PAPER.md:731): the BLS12-381 scalar field r (255 bits, outside the
    reference's q < 2^(bits-4) range) at 256 bits — NTT n=2^16 batch 64
    fwd+inv and vadd/vmul/axpy at n=2^24."""
    from paper_2501_07535_b200 import device as dev
    from paper_2501_07535_b200.params import NttParams
    r = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001
    f = dev.Field(256, r, "montgomery")
    g = 7  # multiplicative generator of F_r
    root = pow(g, (r - 1) // N, r)
    plan = dev.NttPlan(f, NttParams(n=N, p=r, root=root, root_inv=pow(root, -1, r), n_inv=pow(N, -1, r)))
    x = canonical_random(torch, BATCH * N, 555)
    y, z = torch.empty_like(x), torch.empty_like(x)
    ws = torch.empty(plan.workspace_bytes(BATCH) // 4, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()

    def timed(fn, reps=10):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for e0, e1 in evs:
            e0.record(stream)
            fn()
            e1.record(stream)
        torch.cuda.synchronize()
        return statistics.median(a.elapsed_time(b) for a, b in evs)

    ms = timed(lambda: (plan.forward(x, out=y, workspace=ws), plan.inverse(y, out=z, workspace=ws)))
    assert torch.equal(z, x), "full-width NTT roundtrip mismatch"
    res = {"field": "BLS12-381 r (255-bit), 256-bit interface width, Montgomery",
           "ntt_2p16_us_per_transform": round(ms * 1e3 / (2 * BATCH), 3)}
    del x, y, z, ws
    m = 1 << 24
    a = canonical_random(torch, m, 11)
    b = canonical_random(torch, m, 12)
    o = torch.empty_like(a)
    for op in ("vadd", "vmul", "axpy"):
        fn = (lambda: f.axpy(12345, a, b, out=o)) if op == "axpy" else (lambda op=op: getattr(f, op)(a, b, out=o))
        res[f"{op}_2p24_GBps"] = round(3 * 4 * K_LIMBS * m / (timed(fn) * 1e-3) / 1e9, 1)
    del a, b, o
    torch.cuda.empty_cache()
    return res


def run_steady_state(args, torch, plan):
    """The paper's protocol: t_single = t_all / k at
    several batch sizes k, and ns per butterfly = 2 t_single / (n log2 n);
    256-bit n = 2^16 forward + inverse, device-resident."""
    stream = torch.cuda.current_stream()
    rows = []
    for k in (8, 32, 64, 128, 256):
        x = canonical_random(torch, k * N, 31 + k)
        y, z = torch.empty_like(x), torch.empty_like(x)
        ws = torch.empty(plan.workspace_bytes(k) // 4, dtype=torch.int32, device="cuda")
        for _ in range(2):
            plan.forward(x, out=y, workspace=ws)
            plan.inverse(y, out=z, workspace=ws)
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
        for e0, e1 in evs:
            e0.record(stream)
            plan.forward(x, out=y, workspace=ws)
            plan.inverse(y, out=z, workspace=ws)
            e1.record(stream)
        torch.cuda.synchronize()
        ms = statistics.median(a.elapsed_time(b) for a, b in evs)
        t_single = ms * 1e3 / (2 * k)
        rows.append({"batch": k, "us_per_transform": round(t_single, 3),
                     "ns_per_butterfly": round(2 * t_single * 1e3 / (N * LOGN), 5)})
        del x, y, z, ws
    torch.cuda.empty_cache()
    return {"rows": rows, "t_single_us": min(r["us_per_transform"] for r in rows),
            "note": "median of 5; inputs of 8 transforms and up fit in L2 partially (not flushed)"}


def run_batched_2p20(args, torch, rank, world, pg):
    """BASELINE configs[3]: 256-bit NTT n=2^20, batch 256 in total, sharded by
    batch across the ranks (strong scaling, no collective): forward + inverse."""
    from paper_2501_07535_b200 import dist as D
    from paper_2501_07535_b200 import kernels as K
    from paper_2501_07535_b200.params import find_ntt_params
    n, total = 1 << 20, 256
    lo, hi = D.shard_range(total, rank, world)
    b = hi - lo
    plan = K.get_plan(BITS, find_ntt_params(BITS, n))
    x = canonical_random(torch, b * n, 777 + rank)
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    ws = torch.empty(plan.workspace_bytes(b) // 4, dtype=torch.int32, device="cuda")
    plan.forward(x, out=y, workspace=ws)
    plan.inverse(y, out=z, workspace=ws)
    torch.cuda.synchronize()
    assert torch.equal(z, x), "2^20 roundtrip mismatch"
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(pg)
    torch.cuda.synchronize()
    e0.record(stream)
    plan.forward(x, out=y, workspace=ws)
    plan.inverse(y, out=z, workspace=ws)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(pg, e0.elapsed_time(e1))
    del x, y, z, ws
    torch.cuda.empty_cache()
    return {"n": n, "batch_total": total, "ranks": world, "ms_fwd_plus_inv": round(ms, 3),
            "us_per_transform": round(ms * 1e3 / (2 * total), 2), "passes": plan.pass_log_sizes,
            "int_frac_executed": round((plan_work(plan, b, False) + plan_work(plan, b, True)) / (ms * 1e-3)
                                       / int_peak_wmul_per_s()[0], 3),
            "int_frac_reference_work": round(_alg_wmul(n) * 2 * b / (ms * 1e-3) / int_peak_wmul_per_s()[0], 3),
            "int_frac_basis": "word products / time / measured per-GPU product peak (max over ranks' time); "
                              "executed = the plan's own products (wm_ntt_pass_work), reference_work = 3k^2 per "
                              "butterfly (SURVEY.md \u00a78(d); above the executed work)",
            "scaling": "strong (fixed total batch 256)", "note": "max over ranks; inputs 8 GiB / world per rank"}


class _SelfComm:
    def all_to_all(self, out, inp):
        out.copy_(inp)
        return out


def run_reference_gpu(args, torch, plan):
    """The reference's own emit_cuda kernels compiled for sm_100a
    (oracle/_ref/libref_gpu.so, built by oracle/gen_ref.py): vmul at 2^24 and
    the NTT at the largest size that compiles (2^11, 256-bit), beside ours."""
    path = ROOT / "oracle" / "_ref" / "libref_gpu.so"
    if not path.exists():
        return {"unavailable": "oracle/_ref/libref_gpu.so not built"}
    from paper_2501_07535_b200 import device as dev
    from paper_2501_07535_b200 import kernels as K
    from paper_2501_07535_b200.params import find_ntt_params
    lib = ctypes.CDLL(str(path))
    vp, i = ctypes.c_void_p, ctypes.c_int
    stream = torch.cuda.current_stream()
    res = {}

    def timed(fn, reps=10):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    # BLAS 2^24: vadd/vmul/axpy x 128/256/384/768 bits x runtime/baked q, mu
    # in the reference layout (32-bit words MSW first, padded
    # to a power of two), each output checked against ours
    from paper_2501_07535_b200.params import compute_barrett
    n = 1 << 24
    thr = 256
    rows = []
    names = {"vadd": ["a", "b"], "vmul": ["a", "b"], "axpy": ["a", "x", "y"]}
    extra = {"vadd": ["q"], "vmul": ["q", "mu"], "axpy": ["q", "mu"]}

    def words_dev(v, P):
        return torch.tensor([w - (1 << 32) if w >= 1 << 31 else w for w in K.to_words(v, P, 32)],
                            dtype=torch.int32).cuda()

    for bits in args.blas_bits:
        Kl = bits // 32
        P = 1 << (Kl - 1).bit_length()
        q = find_ntt_params(bits, 1).p
        mu = compute_barrett(q, bits).mu
        f = dev.Field(bits, q, "karatsuba" if Kl >= 12 else "schoolbook")
        g = torch.Generator(device="cuda").manual_seed(bits + 5)
        a = torch.randint(-(1 << 31), 1 << 31, (n, Kl), dtype=torch.int32, device="cuda", generator=g)
        b = torch.randint(-(1 << 31), 1 << 31, (n, Kl), dtype=torch.int32, device="cuda", generator=g)
        a[:, Kl - 1] &= (1 << (bits - 5 - 32 * (Kl - 1))) - 1
        b[:, Kl - 1] &= (1 << (bits - 5 - 32 * (Kl - 1))) - 1
        ra, rb = f.to_ref_layout(a, 32, P), f.to_ref_layout(b, 32, P)
        rout = torch.empty_like(ra)
        scal = 123456789
        dv = {"a": ra, "b": rb, "x": ra, "y": rb, "q": words_dev(q, P), "mu": words_dev(mu, P),
              "s": words_dev(scal, P)}
        out = torch.empty_like(a)
        gb = 3 * 4 * Kl * n / 1e9
        for kind in ("vadd", "vmul", "axpy"):
            ours = (lambda: f.axpy(scal, a, b, out=out)) if kind == "axpy" else \
                (lambda kind=kind: getattr(f, kind)(a, b, out=out))
            ms_ours = timed(ours)
            want = out.clone()
            for mode in ("runtime", "baked"):
                name = f"{kind}{n}_{bits}w32_{mode}"
                fn = getattr(lib, "refdrv_" + name, None)
                if fn is None:
                    rows.append({"kind": kind, "bits": bits, "mode": mode, "unavailable": "not built"})
                    continue
                argn = names[kind] + (extra[kind] if mode == "runtime" else [])
                fn.argtypes = [vp] * (len(argn) + 1) + [i, i]
                # axpy's `a` is the scalar: one element in the reference layout
                ptrs = [(dv["s"] if (kind == "axpy" and nm == "a") else dv[nm]).data_ptr() for nm in argn]
                rout.zero_()
                ms_ref = timed(lambda: fn(*ptrs, rout.data_ptr(), n, thr))
                ok = bool(torch.equal(f.from_ref_layout(rout, 32, P), want))
                rows.append({"kind": kind, "bits": bits, "mode": mode, "reference_GBps": round(gb / (ms_ref * 1e-3), 1),
                             "ours_GBps": round(gb / (ms_ours * 1e-3), 1), "speedup": round(ms_ref / ms_ours, 2),
                             "reference_matches_ours": ok})
        del a, b, ra, rb, rout, out, dv
    res["blas_2p24"] = {"rows": rows, "n": n, "ours": "auto reduction (special form), bench strategies",
                        "bytes": "algorithmic 3 x bits/8 per element for both (the reference layout pads "
                                 "384/768-bit values to 16/32 words)",
                        "reference_driver": f"emitted {{kind}}_kernel at {thr} threads/block (its own launcher's "
                                            "1024 threads/block does not launch from 256 bits)"}
    torch.cuda.empty_cache()
    # NTT 2^11 (largest the reference's emitted CUDA compiles at 256 bits), batch 512
    nn, batch = 1 << 11, 512
    prm = find_ntt_params(BITS, nn)
    pl = K.get_plan(BITS, prm)
    x = canonical_random(torch, nn * batch, 13)
    rx = pl.field.to_ref_layout(x, 32, 8)
    ry = torch.empty_like(rx)
    rz = torch.empty_like(rx)
    lib.refdrv_ntt2048_256w32_baked.argtypes = [vp, vp, i, i]
    lib.refdrv_intt2048_256w32_baked.argtypes = [vp, vp, i, i]
    ms_ref = timed(lambda: (lib.refdrv_ntt2048_256w32_baked(rx.data_ptr(), ry.data_ptr(), batch, thr),
                            lib.refdrv_intt2048_256w32_baked(ry.data_ptr(), rz.data_ptr(), batch, thr)), reps=3)
    lib.refdrv_ntt2048_256w32_baked(rx.data_ptr(), ry.data_ptr(), batch, thr)
    torch.cuda.synchronize()
    ok = torch.equal(pl.field.from_ref_layout(ry, 32, 8), pl.forward(x))
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    ms_us = timed(lambda: (pl.forward(x, out=y), pl.inverse(y, out=z)))
    res["ntt_2p11"] = {"batch": batch, "reference_us_per_transform": round(ms_ref * 1e3 / (2 * batch), 3),
                       "ours_us_per_transform": round(ms_us * 1e3 / (2 * batch), 4),
                       "speedup": round(ms_ref / ms_us, 1), "reference_matches_ours": bool(ok),
                       "note": "reference emit_cuda kernels (bit-reverse + one launch per stage, __constant__ "
                               "twiddles) driven at 256 threads/block: its own launcher's 1024 threads/block cannot "
                               "launch at 256 bits; n >= 2^12 does not compile (constant bank overflow)"}
    return res


# ------------------------------------------------------------ CPU baselines
def _ref_lib():
    os.environ.setdefault("OMP_STACKSIZE", "64M")
    # all host cores (torchrun exports OMP_NUM_THREADS=1 to every rank; the
    # reference arm runs on rank 0 alone and should use the whole host)
    os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    path = ROOT / "oracle" / "_ref" / "libref_cpu.so"
    if not path.exists():
        return None
    lib = ctypes.CDLL(str(path))
    try:  # libgomp may have been initialised before we set the variable
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(len(os.sched_getaffinity(0)))
    except OSError:
        pass
    for nm in ("refdrv_ntt65536_256w64", "refdrv_intt65536_256w64"):
        getattr(lib, nm).argtypes = [ctypes.c_void_p, ctypes.c_int64]
    return lib


def cpu_sample_inputs(count: int):
    rng = np.random.Generator(np.random.PCG64(7))
    x = rng.integers(0, 1 << 63, size=(count * N, WORDS64), dtype=np.uint64)
    x[:, 0] &= np.uint64((1 << 59) - 1)  # MSW-first: top word < 2^59 -> value < 2^251 < p
    return np.ascontiguousarray(x)


def run_cpu_reference(transforms: int):
    """The reference's own CPU code (emit_c output, oracle/_ref) on all host
    cores; falls back to the C oracle port when _ref was not built."""
    cores = len(os.sched_getaffinity(0))
    lib = _ref_lib()
    # at least one transform per core in each direction so every core works
    half = max(1, transforms // 2, cores)
    if lib is not None:
        x = cpu_sample_inputs(half)
        y = x.copy()
        t0 = time.perf_counter()
        lib.refdrv_ntt65536_256w64(y.ctypes.data, half)
        lib.refdrv_intt65536_256w64(y.ctypes.data, half)
        dt = time.perf_counter() - t0
        assert np.array_equal(x, y), "reference CPU roundtrip mismatch"
        return {"value": dt * 1e6 / (2 * half), "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": f"{half} forward + {half} inverse 256-bit n=2^16 transforms, reference emit_c "
                          f"(64-bit words, gcc -O2) with OpenMP over transforms"}
    from oracle import bigint
    from oracle.cbind import OracleField
    prm = bigint.find_ntt_params(BITS, N)
    f = OracleField(prm["p"], BITS)
    x = np.random.Generator(np.random.PCG64(7)).integers(0, 1 << 32, size=(half * N, K_LIMBS), dtype=np.uint64)
    x = x.astype(np.uint32)
    x[:, -1] &= (1 << 27) - 1
    t0 = time.perf_counter()
    y = f.ntt(x, N, prm["root"])
    f.ntt(y, N, prm["root_inv"], prm["n_inv"])
    dt = time.perf_counter() - t0
    return {"value": dt * 1e6 / (2 * half), "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{half} forward + {half} inverse transforms, C oracle port (oracle/ntt_oracle.c)"}


def cpu_baseline_subprocess(args):
    """The CPU baseline timed in a fresh process (the --impl reference arm's
    code path): inside this process torch's OpenMP pool, left spinning by the
    earlier host-side tensor work, competes with the reference's OpenMP
    threads for the host cores (1.7x slower measured in-process)."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "3", "--warmup", "1",
           "--ref-transforms", str(2 * max(1, args.cpu_sample // 2))]
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    try:
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
        line = json.loads(res.stdout.strip().splitlines()[-1])
        cb = line["cpu_baseline"]
        cb["process"] = "fresh subprocess (bench.py --impl reference --steps 3 --warmup 1)"
        return cb
    except Exception as exc:  # report, do not fail the bench
        return {"value": None, "unit": UNIT, "cores": None, "kind": "unavailable", "sample": str(exc)[:200]}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _bigint_ntt_job(seed: int) -> float:
    from oracle import bigint
    prm = bigint.find_ntt_params(BITS, N)
    xs = bigint.uniform_residues(np.random.Generator(np.random.PCG64(seed)), N, prm["p"])
    t0 = time.perf_counter()
    bigint.run_ntt(xs, prm, BITS)
    return time.perf_counter() - t0


def run_python_bigint():
    """The reference's Python big-integer run_ntt path (kernels.py:483-499:
    per-butterfly Barrett mulmod/addmod/submod on Python ints), as restated
    line for line by the oracle port (oracle/bigint.run_ntt), on one core
    and fanned out over all host cores with multiprocessing (transforms are
    independent; SURVEY.md §8(d) CPU baseline (i))."""
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    one = _bigint_ntt_job(1)
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(cores) as pool:
        pool.map(_bigint_ntt_job, range(100, 100 + cores))
    wall = time.perf_counter() - t0
    return {"single_process_us_per_transform": round(one * 1e6, 1),
            "all_cores_us_per_transform": round(wall * 1e6 / cores, 1), "cores": cores,
            "sample": f"1 transform on one core; {cores} transforms over {cores} processes (256-bit n=2^16 forward)",
            "kind": "port", "code": "oracle/bigint.run_ntt (line-for-line restatement of the reference run_ntt "
                                    "with its Barrett mulmod; the reference itself is not on the GPU box)"}


def reference_arm(args, rank, world, pg):
    """--impl reference: the reference's CPU implementation of the path."""
    if rank != 0:
        return None
    for _ in range(args.warmup):
        run_cpu_reference(2)
    vals = []
    t_start = time.perf_counter()
    per_step = args.ref_transforms
    for _ in range(args.steps):
        r = run_cpu_reference(per_step)
        vals.append(r["value"])
    wall = time.perf_counter() - t_start
    value = statistics.mean(vals)
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall * 1e3 / args.steps, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": "256-bit forward+inverse NTT n=2^16 batch 64 (BASELINE configs[1]); --ref-transforms per step, default the whole 64+64 step",
                   "bits": BITS, "n": N, "transforms_per_step": 2 * (per_step // 2)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
                         "sample": r["sample"], "cpu_model": cpu_model(),
                         "python_bigint": run_python_bigint() if args.python_bigint else None},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# ------------------------------------------------------------ main
_JSON_OUT = None


def emit(obj) -> None:
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(obj) + "\n")
    out.flush()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-transforms", type=int, default=2 * BATCH,
                    help="transforms per reference-arm step (default: the whole 64 fwd + 64 inv step)")
    ap.add_argument("--cpu-sample", type=int, default=2 * BATCH,
                    help="transforms per CPU-baseline step (default: the whole batch-64 fwd+inv step)")
    ap.add_argument("--skip-extras", action="store_true", help="only the headline workload")
    ap.add_argument("--python-bigint", type=int, default=1,
                    help="reference arm: also time the Python big-int run_ntt path (1/0)")
    ap.add_argument("--extras", nargs="*", default=list(EXTRAS), choices=list(EXTRAS),
                    help="which extra measurements to run (default: all)")
    ap.add_argument("--blas-bits", type=int, nargs="*", default=[128, 256, 384, 768])
    ap.add_argument("--e2e-chunk", type=int, default=0, help="transforms per host-pipeline chunk (0 = auto)")
    ap.add_argument("--dist-backend", default="auto", choices=["auto", "nccl", "gloo"],
                    help="N>1 process group: nccl (one GPU per rank) or gloo (dry run, ranks may share a GPU)")
    args = ap.parse_args()
    # stdout carries exactly one JSON line: anything libraries print there
    # (NCCL prints its version banner to stdout) goes to stderr instead
    sys.stdout.flush()
    global _JSON_OUT
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    if args.warmup < 3 and args.impl == "ours":
        log("note: warmup < 3 raised to 3")
        args.warmup = 3

    rank, world, local, pg = dist_setup(args.gpus, args.dist_backend)
    if args.impl == "reference":
        out = reference_arm(args, rank, world, pg)
        if rank == 0:
            emit(out)
        if pg is not None:
            pg.destroy_process_group()
        return

    res = run_gpu(args, rank, world, local, pg)
    if rank != 0:
        if pg is not None:
            pg.barrier()
            pg.destroy_process_group()
        return

    # roofline of the dominant kernel: ntt_col_pass (pass 0), integer pipe.
    # achieved = word products the launch executes (wm_ntt_pass_work) / its
    # event-timed duration; peak = this run's measured product throughput.
    sizes = res["pass_log_sizes"]
    peak, _ = int_peak_wmul_per_s()
    pass_ms = res["pass0_ms"]
    muls, wprod = res["pass0_work"]
    achieved = wprod / (pass_ms * 1e-3)
    bflies = BATCH * (N // 2) * sizes[0]  # one pass = log2(L) radix-2 stages over the batch
    ref_achieved = bflies * ALG_WMUL_PER_BFLY / (pass_ms * 1e-3)
    kname = f"ntt_col_pass<8, {res['plan_mode']}>"
    traffic = None
    pipes = None
    try:
        prof = json.loads((ROOT / "profiles" / "r02_ncu_traffic.json").read_text())
        kp = prof[kname]
        traffic = kp["dram_bytes_per_launch"]
        pipes = {"fmaheavy_pct": kp.get("fmaheavy_pct"), "alu_pct": kp.get("alu_pct"),
                 "basis": "ncu --set full of the same kernel (profiles/r02_ncu_traffic.json)"}
    except Exception:
        pass
    roofline = {
        "bound": "int", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "T word-products/s",
        "frac": achieved / peak, "traffic": traffic,
        "kernel": f"{kname} (pass 0 of {'+'.join('2^%d' % s for s in sizes)}), batch 64, "
                  f"{pass_ms * 1e3:.1f} us/launch",
        "work": f"{muls} field multiplications x {wprod / max(1, muls):.0f} word products (32x32->64) each = "
                f"{wprod:.4g} per launch, as executed (wm_ntt_pass_work; two-fold special-form products)",
        "peak_basis": "32x32->64 products/s measured in this run by wm_probe_imad_wide (best of mad.wide/"
                      f"mul.wide chains at full occupancy: {INT_PEAK.get('mul_wide_per_s', 0) / 1e12:.3f} / "
                      f"{INT_PEAK.get('mad_wide_per_s', 0) / 1e12:.3f} T/s)",
        "reference_work_basis": {"achieved": ref_achieved / 1e12, "frac": ref_achieved / peak,
                                 "work": f"{ALG_WMUL_PER_BFLY} products per butterfly (reference 3k^2, SURVEY.md "
                                         f"\u00a78(d)) x {bflies} butterflies",
                                 "note": "the reference algorithm's products; the kernel executes fewer, so this "
                                         "fraction can exceed 1"},
        "traffic_basis": "dram__bytes_read+write per launch, ncu --set full (profiles/r02_ncu_traffic.json); "
                         "algorithmic bytes per launch = 2 x 128 MiB",
        "ns_per_butterfly_paper_metric": 2 * (res["ms_per_step"] * 1e6 / (2 * BATCH)) / (N * LOGN),
        "pipe_utilisation": pipes,
    }
    # the CPU baseline once, on rank 0, after every rank's GPU work (the other
    # ranks wait at the final barrier)
    cpu = cpu_baseline_subprocess(args)
    out = {
        "metric": METRIC,
        "value": res["us_per_transform"],
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": res["ms_per_step"],
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic",
        "config": {"workload": "256-bit forward+inverse NTT n=2^16 batch 64 per GPU (BASELINE configs[1])",
                   "bits": BITS, "n": N, "batch_per_gpu": BATCH, "transforms_per_step": 2 * BATCH,
                   "parallelism": f"batch-sharded x{world}", "l2": "flushed between timed steps (252 MiB write)",
                   "reduction": f"{res['reduction']} (p = 2^252 - c, c < 2^32: two-fold products; "
                                "headline_generic_barrett = the same step on the generic path)",
                   "dist_backend": DIST["backend"],
                   "passes": sizes},
        "e2e": res["e2e"],
        "gpu_launches": res["launches_per_step"] * args.steps,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": res["clocks"],
        "int_peak_measured": {k: round(v / 1e12, 4) for k, v in INT_PEAK.items()},
        "reduction": res["reduction"],
        "headline_generic_barrett": res["generic"],
        "blas": res["blas"],
        "four_step_2p24": res["four_step"],
        "batched_2p20_x256": res["batched_2p20"],
        "reference_gpu": res["reference_gpu"],
        "full_width_bls12_381": res["full_width"],
        "steady_state_2p16": res["steady_state"],
        "drop_in_host_boundary": res["drop_in"],
    }
    emit(out)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
