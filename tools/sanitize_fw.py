"""Small full-width workloads for compute-sanitizer (Montgomery and Shoup/[0,4p) NTT modes, BLAS, dist scatter)."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2501_07535_b200 import device as dev, dist as D
from paper_2501_07535_b200.params import NttParams
for p, g in ((0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001, 7),
             (21888242871839275222246405745257275088548364400416034343698204186575808495617, 5)):
    for logn in (10, 18):
        n = 1 << logn
        w = pow(g, (p - 1) // n, p)
        prm = NttParams(n=n, p=p, root=w, root_inv=pow(w, -1, p), n_inv=pow(n, -1, p))
        f = dev.Field(256, p, "montgomery")
        plan = dev.NttPlan(f, prm)
        x = torch.randint(0, 1 << 28, (2 * n, 8), dtype=torch.int32, device="cuda")
        assert torch.equal(plan.inverse(plan.forward(x)), x)
        f.vmul(x, x); f.axpy(3, x, x); f.vadd(x, x)
    engines = [D.FourStepNtt(256, NttParams(n=1 << 12, p=p, root=pow(g, (p - 1) >> 12, p),
                                            root_inv=pow(pow(g, (p - 1) >> 12, p), -1, p), n_inv=pow(1 << 12, -1, p)),
                             k, 2, strategy="montgomery") for k in range(2)]
    xs = [torch.randint(0, 1 << 28, (32, 64, 8), dtype=torch.int32, device="cuda") for _ in range(2)]
    D.loopback_transform_fused(engines, xs)
torch.cuda.synchronize()
print("done")
