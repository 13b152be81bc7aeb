"""Full-output checksums of BASELINE configs 2, 4 and 5 from the pinned C
oracle (oracle/ntt_oracle.c: the reference's run_ntt, kernels.py:483-499,
with the reference's own Barrett constants; pinned equal to the reference's
run_ntt at 2^16 in tests/test_oracle_pinned.py).  Writes
tests/golden/ntt_configs.json; the GPU tests (tests/test_configs_gpu.py)
must match every hash.

    python tests/golden/make_ntt_configs.py      (~1 min on 8 cores)

Inputs: oracle.bigint.uniform_residue_limbs(PCG64(seed)) — uniform canonical
residues.  Hashes are SHA-256 of the little-endian uint32
limbs [batch * n, 8] (element after element, transform after transform).
Forward rows hash NTT(x); inverse rows hash INTT(x) of the same x (an
independent check of the inverse path, not the round trip).
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle import bigint  # noqa: E402
from oracle.cbind import OracleField  # noqa: E402

CONFIGS = [
    # (name, bits, log2 n, batch, seed)
    ("cfg2_2p16_x64", 256, 16, 64, 2),
    ("cfg4_2p20_x4", 256, 20, 4, 4),
    ("cfg5_2p24", 256, 24, 1, 5),
]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u4").tobytes()).hexdigest()


def main():
    rows = []
    for name, bits, logn, batch, seed in CONFIGS:
        n = 1 << logn
        prm = bigint.find_ntt_params(bits, n)
        p = prm["p"]
        t0 = time.time()
        x = bigint.uniform_residue_limbs(np.random.Generator(np.random.PCG64(seed)), batch * n, p)
        of = OracleField(p, bits)
        fwd = of.ntt(x, n, prm["root"])
        inv = of.ntt(x, n, prm["root_inv"], prm["n_inv"])
        per = n * x.shape[1]
        rows.append({
            "name": name, "bits": bits, "n": n, "batch": batch, "seed": seed, "p": str(p),
            "generator": "oracle.bigint.uniform_residue_limbs(PCG64(seed))",
            "x_sha256": sha(x), "fwd_sha256": sha(fwd), "inv_sha256": sha(inv),
            # per-transform hashes localise a mismatch to one transform
            "fwd_sha256_each": [sha(fwd.reshape(-1)[b * per:(b + 1) * per]) for b in range(batch)],
            "inv_sha256_each": [sha(inv.reshape(-1)[b * per:(b + 1) * per]) for b in range(batch)],
            "fwd_head": [str(v) for v in bigint_head(fwd)],
        })
        print(f"{name}: {time.time() - t0:.1f} s", flush=True)
    (HERE / "ntt_configs.json").write_text(json.dumps(rows, indent=1) + "\n")


def bigint_head(a: np.ndarray, count: int = 4):
    return [int.from_bytes(np.ascontiguousarray(a[i]).tobytes(), "little") for i in range(count)]


if __name__ == "__main__":
    main()
