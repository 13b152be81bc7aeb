"""Full-width (Montgomery) fields: BLS12-381 scalar-field NTT (n=2^16, batch
64, fwd+inv) and 256-bit vmul/axpy GB/s, beside the reference-range fields."""
import json, statistics, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2501_07535_b200 import device as dev, kernels as K
from paper_2501_07535_b200.params import NttParams, find_ntt_params

R = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001

def t(fn, reps=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)

def params(p, n):
    x = 2
    while pow(x, (p - 1) // 2, p) != p - 1: x += 1
    r = pow(x, (p - 1) // n, p)
    return NttParams(n=n, p=p, root=r, root_inv=pow(r, -1, p), n_inv=pow(n, -1, p))

def main():
    out = {}
    n, B = 1 << 16, 64
    f = dev.Field(256, R, "montgomery")
    plan = dev.NttPlan(f, params(R, n))
    x = torch.randint(0, 1 << 30, (B * n, 8), dtype=torch.int32, device="cuda")
    x[:, 7] &= (1 << 29) - 1
    y = torch.empty_like(x); z = torch.empty_like(x)
    ws = torch.empty(plan.workspace_bytes(B) // 4, dtype=torch.int32, device="cuda")
    ms = t(lambda: (plan.forward(x, out=y, workspace=ws), plan.inverse(y, out=z, workspace=ws)))
    assert torch.equal(z, x)
    out["bls12_381_r_ntt_2p16_us_per_transform"] = round(ms * 1e3 / (2 * B), 3)
    BN = 21888242871839275222246405745257275088548364400416034343698204186575808495617
    fb = dev.Field(256, BN, "montgomery")
    pb = dev.NttPlan(fb, params(BN, n))
    msb = t(lambda: (pb.forward(x, out=y, workspace=ws), pb.inverse(y, out=z, workspace=ws)))
    assert torch.equal(z, x)
    out["bn254_r_ntt_2p16_us_per_transform"] = round(msb * 1e3 / (2 * B), 3)
    ref = K.get_plan(256, find_ntt_params(256, n))
    ms2 = t(lambda: (ref.forward(x, out=y, workspace=ws), ref.inverse(y, out=z, workspace=ws)))
    out["reference_range_ntt_2p16_us_per_transform"] = round(ms2 * 1e3 / (2 * B), 3)
    m = 1 << 24
    a = torch.randint(0, 1 << 30, (m, 8), dtype=torch.int32, device="cuda"); a[:, 7] &= (1 << 29) - 1
    b = a.flip(0).contiguous(); o = torch.empty_like(a)
    for op in ("vadd", "vmul", "axpy"):
        fn = (lambda: f.axpy(12345, a, b, out=o)) if op == "axpy" else (lambda op=op: getattr(f, op)(a, b, out=o))
        out[f"bls12_381_r_{op}_2p24_GBps"] = round(96 * m / t(fn) / 1e6, 1)
    print(json.dumps(out))

main()
