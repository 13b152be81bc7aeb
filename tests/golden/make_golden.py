"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
package itself (/root/reference/pkg/src/widemod) — its own parameter search,
its own lowered kernels (generate_kernel -> compile_program) and executors
(run_vector / run_ntt).  Run in the build container only (the reference does
not exist on the GPU box); the JSON it writes is committed.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parent.parent))

from widemod.kernels import (  # noqa: E402  (reference package)
    build_program, generate_kernel, make_spec, run_ntt, run_vector, twiddle_table,
)
from widemod.ir import compile_program  # noqa: E402
from widemod.oracle import compute_barrett, find_ntt_params  # noqa: E402

from oracle.bigint import uniform_residues  # noqa: E402


def limbs_sha256(values, K):
    buf = b"".join(int(v).to_bytes(4 * K, "little") for v in values)
    return hashlib.sha256(buf).hexdigest()


def params_fixture():
    rows = []
    cases = [(8, 1), (8, 4), (16, 1), (16, 4), (16, 8), (16, 16), (16, 32), (16, 64),
             (32, 1), (32, 16), (64, 1), (64, 16), (128, 1), (128, 16), (128, 1024),
             (256, 1), (256, 16), (256, 1024), (256, 1 << 16), (256, 1 << 20), (256, 1 << 24),
             (384, 1), (384, 64), (384, 1 << 16), (768, 1), (768, 16), (768, 1 << 10),
             (1024, 4)]
    for width, n in cases:
        t0 = time.time()
        p = find_ntt_params(width, n)
        b = compute_barrett(p.p, width)
        rows.append({"width": width, "n": n, "p": str(p.p), "root": str(p.root),
                     "root_inv": str(p.root_inv), "n_inv": str(p.n_inv),
                     "mu": str(b.mu), "mbits": b.mbits, "shift1": b.shift1, "shift2": b.shift2})
        print(f"params {width} {n}: {time.time() - t0:.2f}s", flush=True)
    return rows


def blas_fixture():
    rows = []
    for bits, word, n in [(16, 8, 40), (13, 8, 16), (64, 64, 40), (128, 64, 40), (256, 64, 40),
                          (256, 32, 16), (384, 64, 24), (768, 64, 12)]:
        for kind in ("vadd", "vsub", "vmul", "axpy"):
            spec = make_spec(kind, bits, word, size=n + 9 if kind != "axpy" else n)
            prog = generate_kernel(spec)
            q = spec.barrett.q
            rnd = random.Random(1000 + bits + n)
            if kind == "axpy":
                xs = [rnd.randrange(q) for _ in range(n)]
                ys = [rnd.randrange(q) for _ in range(n)]
                s = rnd.randrange(q)
                out = run_vector(prog, s, xs, ys)
                rows.append({"kind": kind, "bits": bits, "word": word, "q": str(q), "scalar": str(s),
                             "a": [str(x) for x in xs], "b": [str(y) for y in ys],
                             "out": [str(o) for o in out]})
            else:
                edge = (0, 1, q - 1)
                xs = [a for a in edge for _ in edge] + [rnd.randrange(q) for _ in range(n)]
                ys = [b for _ in edge for b in edge] + [rnd.randrange(q) for _ in range(n)]
                out = run_vector(prog, xs, ys)
                rows.append({"kind": kind, "bits": bits, "word": word, "q": str(q),
                             "a": [str(x) for x in xs], "b": [str(y) for y in ys],
                             "out": [str(o) for o in out]})
            print(f"blas {kind} {bits}w{word}", flush=True)
    return rows


def ntt_fixture():
    rows = []
    for bits, word, n in [(16, 8, 4), (16, 8, 8), (16, 8, 64), (64, 64, 16), (128, 64, 16),
                          (128, 64, 256), (256, 64, 16), (256, 64, 1024), (384, 64, 64),
                          (768, 64, 16)]:
        fwd = generate_kernel(make_spec("ntt", bits, word, size=n))
        inv = generate_kernel(make_spec("intt", bits, word, size=n))
        p = int(fwd.attributes["p"])
        rnd = random.Random(77 + bits + n)
        for v in range(2):
            vec = [rnd.randrange(p) for _ in range(n)]
            yf = run_ntt(fwd, vec)
            yi = run_ntt(inv, vec)
            rows.append({"bits": bits, "word": word, "n": n, "p": str(p),
                         "x": [str(a) for a in vec], "fwd": [str(a) for a in yf],
                         "inv": [str(a) for a in yi]})
        print(f"ntt {bits}w{word} n={n}", flush=True)
    return rows


def ntt_large_fixture():
    """256-bit n=2^16 through the reference's unlowered program (its big-int
    executor): inputs regenerated from PCG64(seed) by oracle.bigint.uniform_residues."""
    rows = []
    n = 1 << 16
    fwd = build_program(make_spec("ntt", 256, 64, size=n))
    inv = build_program(make_spec("intt", 256, 64, size=n))
    ffn, ifn = compile_program(fwd), compile_program(inv)
    p = int(fwd.attributes["p"])
    for seed in (0, 1):
        vec = uniform_residues(np.random.Generator(np.random.PCG64(seed)), n, p)
        t0 = time.time()
        yf = run_ntt(fwd, vec, fn=ffn)
        yi = run_ntt(inv, vec, fn=ifn)
        rows.append({"bits": 256, "n": n, "p": str(p), "seed": seed, "generator": "uniform_residues/PCG64",
                     "x_sha256": limbs_sha256(vec, 8), "fwd_sha256": limbs_sha256(yf, 8),
                     "inv_sha256": limbs_sha256(yi, 8), "fwd_head": [str(a) for a in yf[:4]],
                     "inv_head": [str(a) for a in yi[:4]]})
        print(f"ntt 2^16 seed {seed}: {time.time() - t0:.1f}s", flush=True)
    return rows


def butterfly_fixture():
    """run_program on transform kinds: the reference's lowered butterfly
    (build_ntt, kernels.py:270-311) on (u, v, w) operands, edge values included."""
    from widemod.kernels import run_program
    rows = []
    for bits, word, n in [(16, 8, 8), (64, 64, 16), (128, 64, 16), (256, 64, 1024), (256, 32, 16),
                          (384, 64, 64), (768, 64, 16)]:
        for kind in ("ntt", "intt"):
            prog = generate_kernel(make_spec(kind, bits, word, size=n))
            p = int(prog.attributes["p"])
            rnd = random.Random(5 + bits + n)
            edge = (0, 1, p - 1)
            ops = [(u, v, w) for u in edge for v in edge for w in edge]
            ops += [(rnd.randrange(p), rnd.randrange(p), rnd.randrange(p)) for _ in range(12)]
            outs = [run_program(prog, u, v, w) for u, v, w in ops]
            rows.append({"kind": kind, "bits": bits, "word": word, "n": n, "p": str(p),
                         "ops": [[str(a) for a in t] for t in ops],
                         "out": [[str(a) for a in o] for o in outs]})
        print(f"butterfly {bits}w{word}", flush=True)
    return rows


def twiddle_fixture():
    rows = []
    for width, n in [(16, 8), (128, 16), (256, 1024)]:
        prm = find_ntt_params(width, n)
        rows.append({"width": width, "n": n, "fwd": [str(x) for x in twiddle_table(prm)],
                     "inv": [str(x) for x in twiddle_table(prm, inverse=True)]})
    return rows


def main():
    which = sys.argv[1:] or ["params", "blas", "ntt", "ntt_large", "twiddles", "butterfly"]
    makers = {"params": params_fixture, "blas": blas_fixture, "ntt": ntt_fixture,
              "ntt_large": ntt_large_fixture, "twiddles": twiddle_fixture, "butterfly": butterfly_fixture}
    for name in which:
        data = makers[name]()
        (HERE / f"{name}.json").write_text(json.dumps(data, indent=0, sort_keys=True) + "\n")
        print(f"wrote {name}.json")


if __name__ == "__main__":
    main()
