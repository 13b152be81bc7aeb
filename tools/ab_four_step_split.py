"""A/B of the four-step split at one rank (256-bit n = 2^24): forward time of
FourStepNtt for several (N1, N2), each checked against the single-GPU plan
(gather of the one-rank output = natural-order NTT).

    python tools/ab_four_step_split.py
"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2501_07535_b200 import dist as D
from paper_2501_07535_b200 import kernels as K
from paper_2501_07535_b200.params import find_ntt_params


class SelfComm:
    def all_to_all(self, out, inp):
        out.copy_(inp)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)


n = 1 << 24
prm = find_ntt_params(256, n)
plan = K.get_plan(256, prm)
g = torch.Generator(device="cuda").manual_seed(5)
xs = torch.randint(0, 1 << 27, (n, 8), dtype=torch.int32, device="cuda", generator=g)
ref = plan.forward(xs)
torch.cuda.synchronize()
res = {"single_plan_ms": round(timed(lambda: plan.forward(xs)), 4), "default_split": D.split_lengths(n)}
for n1 in (1 << 12, 1 << 14, 1 << 16, 1 << 15, 1 << 13):
    n2 = n // n1
    eng = D.FourStepNtt(256, prm, 0, 1, comm=SelfComm(), split=(n1, n2))
    x = eng.layout.scatter_input(xs, 0)
    y = eng.forward(x)
    ok = torch.equal(y.transpose(0, 1).reshape(n, 8), ref)  # rows k2 of y[k2 + N2 k1]
    res[f"{n1}x{n2}"] = {"ms": round(timed(lambda: eng.forward(x)), 4), "passes": [eng.backend.plan_n2.pass_log_sizes,
                         eng.backend.plan_n1.pass_log_sizes], "matches_plan": bool(ok)}
    del eng, x, y
    torch.cuda.empty_cache()
print(json.dumps(res))

# phase breakdown of the default split (NCCL-form pipeline at one rank)
eng = D.FourStepNtt(256, prm, 0, 1, comm=SelfComm())
x = eng.layout.scatter_input(xs, 0)
L = eng.layout
b = eng.backend
y1 = b.row_ntt(x, L.n2, False)
c = b.scale_transpose(y1, False)
d = torch.empty_like(c)
e = b.block_transpose(d, 1, L.n2, L.n1)
br = {"row_ntt_n2_ms": timed(lambda: b.row_ntt(x, L.n2, False)),
      "scale_transpose_ms": timed(lambda: b.scale_transpose(y1, False)),
      "a2a_copy_ms": timed(lambda: d.copy_(c)),
      "block_transpose_ms": timed(lambda: b.block_transpose(d, 1, L.n2, L.n1)),
      "row_ntt_n1_ms": timed(lambda: b.row_ntt(e, L.n1, False)),
      "total_ms": timed(lambda: eng.forward(x))}
print(json.dumps({f"breakdown_{L.n1}x{L.n2}": {k: round(v, 4) for k, v in br.items()}}))
