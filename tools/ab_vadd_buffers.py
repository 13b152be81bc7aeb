"""128-bit vadd, ours vs the reference's emitted kernel, each timed on BOTH
buffer sets (ours' limb tensors and the reference-layout copies): separates
the kernels from where their operands happen to sit in HBM."""
import ctypes, json, statistics, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2501_07535_b200 import device as dev
from paper_2501_07535_b200.params import find_ntt_params
ROOT = Path(__file__).resolve().parent.parent
lib = ctypes.CDLL(str(ROOT / "oracle/_ref/libref_gpu.so"))
fn = lib.refdrv_vadd16777216_128w32_baked
fn.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_int]
def timed(f, reps=30):
    for _ in range(3): f()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(); f(); b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)
n = 1 << 24
q = find_ntt_params(128, 1).p
fld = dev.Field(128, q)
a = torch.randint(0, 1 << 27, (n, 4), dtype=torch.int32, device="cuda"); b = a.flip(0).contiguous(); o = torch.empty_like(a)
ra, rb = fld.to_ref_layout(a, 32, 4), fld.to_ref_layout(b, 32, 4); ro = torch.empty_like(ra)
gb = 48 * n / 1e9
res = {}
for rep in range(3):
    for name, (x, y, z) in (("set_ours", (a, b, o)), ("set_ref", (ra, rb, ro))):
        res.setdefault(f"ours_on_{name}", []).append(gb / timed(lambda: fld.vadd(x, y, out=z)) * 1e3)
        res.setdefault(f"ref_on_{name}", []).append(gb / timed(lambda: fn(x.data_ptr(), y.data_ptr(), z.data_ptr(), n, 256)) * 1e3)
print(json.dumps({k: [round(v, 1) for v in vs] for k, vs in res.items()}))
