"""BASELINE configs 2, 4 and 5 pinned hash for hash (tests/golden/ntt_configs.json,
made by tests/golden/make_ntt_configs.py from the pinned C oracle): every
output element of the 256-bit NTT at n = 2^16 x 64, 2^20 x 4 and 2^24, both
directions, through the single-GPU plan (out of place, in place, caller
workspace, plan workspace) and through the distributed four-step engine over
P = 2/4/8 virtual ranks (both exchange forms) after gather_output.  Also
run_program on transform kinds against the reference's own butterfly
(tests/golden/butterfly.json).  Bit-exact (integer work)."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from oracle import bigint

pytestmark = pytest.mark.gpu


def _sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u4").tobytes()).hexdigest()


def _row(golden, name):
    return next(r for r in golden("ntt_configs") if r["name"] == name)


def _inputs(row):
    x = bigint.uniform_residue_limbs(np.random.Generator(np.random.PCG64(row["seed"])),
                                     row["batch"] * row["n"], int(row["p"]))
    assert _sha(x) == row["x_sha256"]
    return x


def _plan(n):
    from paper_2501_07535_b200 import kernels as K
    from paper_2501_07535_b200.params import find_ntt_params
    return K.get_plan(256, find_ntt_params(256, n))


def _check(got: np.ndarray, row, which: str):
    if _sha(got) == row[f"{which}_sha256"]:
        return
    per = row["n"] * 8
    flat = got.reshape(-1)
    bad = [b for b in range(row["batch"])
           if _sha(flat[b * per:(b + 1) * per]) != row[f"{which}_sha256_each"][b]]
    raise AssertionError(f"{row['name']} {which}: transforms {bad[:8]} differ from the oracle")


@pytest.mark.parametrize("name", ["cfg2_2p16_x64", "cfg4_2p20_x4", "cfg5_2p24"])
def test_config_hashes_single_gpu(cuda, golden, name):
    import torch
    from paper_2501_07535_b200 import device as dev
    row = _row(golden, name)
    plan = _plan(row["n"])
    x = _inputs(row)
    xd = dev.to_device(x)
    _check(dev.to_host(plan.forward(xd)), row, "fwd")
    _check(dev.to_host(plan.inverse(xd)), row, "inv")
    # in place with a caller workspace, then the plan's own workspace on a side stream
    ws = torch.empty(max(1, plan.workspace_bytes(row["batch"]) // 4), dtype=torch.int32, device="cuda")
    y = xd.clone()
    plan.forward(y, out=y, workspace=ws)
    _check(dev.to_host(y), row, "fwd")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        z = plan.inverse(xd, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    _check(dev.to_host(z), row, "inv")


@pytest.mark.parametrize("P", [2, 4, 8])
def test_config5_four_step_loopback(cuda, golden, P):
    """Config 5 through the distributed engine: P virtual ranks on one GPU,
    gathered output hash-equal to the oracle; the inverse maps the output
    distribution back (INTT of the same x, gathered in input order)."""
    import torch
    from paper_2501_07535_b200 import device as dev
    from paper_2501_07535_b200 import dist as D
    from paper_2501_07535_b200.params import find_ntt_params
    row = _row(golden, "cfg5_2p24")
    n = row["n"]
    prm = find_ntt_params(256, n)
    engines = [D.FourStepNtt(256, prm, r, P) for r in range(P)]
    L = engines[0].layout
    x = dev.to_device(_inputs(row))
    xs = [L.scatter_input(x, r) for r in range(P)]
    for fused in (False, True):
        ys = (D.loopback_transform_fused if fused else D.loopback_transform)(engines, xs)
        y = L.gather_output([dev.to_host(t) for t in ys])
        _check(y, row, "fwd")
        del ys, y
    # inverse of x: feed x in the OUTPUT distribution, gather in input order
    xo = [L.scatter_output(x, r) for r in range(P)]
    zs = D.loopback_transform(engines, xo, inverse=True)
    _check(L.gather_input([dev.to_host(t) for t in zs]), row, "inv")
    del engines, xs, xo, zs
    torch.cuda.empty_cache()


def test_run_program_butterfly_matches_reference(cuda, golden):
    """run_program on "ntt"/"intt" kinds is the reference's butterfly
    (u + v w, u - v w) mod p (kernels.py:270-311, 442-464)."""
    from paper_2501_07535_b200 import kernels as K
    for row in golden("butterfly"):
        prog = K.generate_kernel(K.make_spec(row["kind"], row["bits"], row["word"], size=row["n"]))
        for ops, want in zip(row["ops"], row["out"]):
            got = K.run_program(prog, *[int(v) for v in ops])
            assert tuple(got) == tuple(int(v) for v in want), (row["bits"], row["kind"], ops)
