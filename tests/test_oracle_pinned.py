"""Pin the oracle (test infrastructure) before trusting it: every known-answer
value from the reference's own tests for the hot path, plus the golden
fixtures tests/golden/*.json that make_golden.py produced by running the
reference package itself."""

from __future__ import annotations

import hashlib
import random

import numpy as np
import pytest

from oracle import bigint
from oracle.cbind import OracleField


def limbs(values, K):
    buf = b"".join(int(v).to_bytes(4 * K, "little") for v in values)
    return np.frombuffer(buf, dtype="<u4").reshape(-1, K).copy()


def ints(arr):
    return [int.from_bytes(r.tobytes(), "little") for r in np.ascontiguousarray(arr, dtype="<u4")]


# ---- reference tests/test_oracle.py pins
def test_modop_pins():  # test_oracle.py:25-29
    assert bigint.modop("add", 7, 9, 13) == 3
    assert bigint.modop("mul", 1, 4092, 4093) == 4092
    assert bigint.modop("sub", 3, 5, 13) == 11
    assert bigint.modop("pow", 5, 4, 13) == 1


def test_barrett_pins():  # test_oracle.py:54-65
    assert bigint.compute_barrett(13, 8) == (4, 157, 2, 9)
    mbits, mu, s1, s2 = bigint.compute_barrett(4093, 16)
    assert (mbits, mu, s1, s2) == (12, 32792, 10, 17)


def test_barrett_exhaustive_q13():  # test_oracle.py:78-82
    for a in range(13):
        for b in range(13):
            assert bigint.barrett_mulmod(a, b, 13, 8) == a * b % 13


@pytest.mark.parametrize("width", [8, 16, 32, 64, 128, 256, 384, 768])
def test_barrett_one_subtraction_enough(width):
    """The reference claims one conditional subtraction always suffices
    (oracle.py:137-149): if it did not, its outputs would be non-canonical
    and could not equal an exact device result."""
    rnd = random.Random(width)
    lo, hi = 1 << (width - 5), 1 << (width - 4)
    for _ in range(300):
        q = rnd.randrange(lo + 1, hi)
        a, b = rnd.randrange(q), rnd.randrange(q)
        assert bigint.barrett_mulmod(a, b, q, width) == a * b % q
        assert bigint.barrett_mulmod(q - 1, q - 1, q, width) == (q - 1) ** 2 % q


def test_is_prime_pins():  # test_oracle.py:96-112
    for n in range(2, 100):
        assert bigint.is_prime(n) == all(n % d for d in range(2, n))
    assert not bigint.is_prime(561)
    assert not bigint.is_prime(341550071728321)
    assert bigint.is_prime((1 << 61) - 1)
    assert bigint.is_prime((1 << 89) - 1)
    assert not bigint.is_prime(((1 << 89) - 1) * ((1 << 61) - 1))


def test_find_ntt_params_pins():  # test_oracle.py:115-137
    assert bigint.find_ntt_params(8, 4) == {"n": 4, "p": 13, "root": 5, "root_inv": 8, "n_inv": 10}
    for n, p in [(1, 4093), (8, 4073), (16, 4049), (32, 4001), (64, 3457)]:
        assert bigint.find_ntt_params(16, n)["p"] == p
    assert bigint.find_ntt_params(64, 1)["p"] == 1152921504606846883


def test_params_golden(golden):
    for row in golden("params"):
        if row["n"] > 1 << 16:
            continue  # the big root scans are covered by test_params.py on the product
        got = bigint.find_ntt_params(row["width"], row["n"])
        assert got["p"] == int(row["p"]) and got["root"] == int(row["root"])
        assert got["root_inv"] == int(row["root_inv"]) and got["n_inv"] == int(row["n_inv"])
        mbits, mu, s1, s2 = bigint.compute_barrett(got["p"], row["width"])
        assert (mu, mbits, s1, s2) == (int(row["mu"]), row["mbits"], row["shift1"], row["shift2"])


def test_convolve_pins():  # test_oracle.py:160-163
    assert bigint.convolve_mod([1, 0, 0, 0], [5, 6, 7, 8], 13) == [5, 6, 7, 8]
    assert bigint.convolve_mod([1, 1, 0, 0], [1, 1, 0, 0], 13) == [1, 2, 1, 0]


# ---- reference tests/test_kernels.py pins
def test_scalar_pins():  # test_kernels.py:82-90 (q=500 at width 13; q=4093 at 16)
    assert bigint.addmod(300, 400, 500) == 200
    assert bigint.submod(100, 300, 500) == 300
    assert bigint.barrett_mulmod(3000, 2000, 4093, 16) == 3755


def test_vector_pins():  # test_kernels.py:113-120
    assert bigint.run_vector("vadd", 500, 13, [300, 499, 0, 250], [400, 1, 0, 250]) == [200, 0, 0, 0]
    assert bigint.run_vector("axpy", 500, 13, 0, [5, 6, 7], [9, 8, 7]) == [9, 8, 7]
    assert bigint.run_vector("vmul", 500, 13, [1, 1, 1], [123, 456, 499]) == [123, 456, 499]


def test_twiddle_pins(golden):  # test_kernels.py:147-153
    assert bigint.twiddle_table(13, 4, 5) == [1, 5]
    assert bigint.twiddle_table(17, 8, 2) == [1, 2, 4, 8]
    assert bigint.twiddle_table(17, 8, 9) == [1, 9, 13, 15]
    for row in golden("twiddles"):
        prm = bigint.find_ntt_params(row["width"], row["n"])
        assert bigint.twiddle_table(prm["p"], row["n"], prm["root"]) == [int(x) for x in row["fwd"]]
        assert bigint.twiddle_table(prm["p"], row["n"], prm["root_inv"]) == [int(x) for x in row["inv"]]


def test_ntt_pins():  # test_kernels.py:156-161
    prm = bigint.find_ntt_params(8, 4)
    assert bigint.run_ntt([1, 0, 0, 0], prm, 8) == [1, 1, 1, 1]
    assert bigint.run_ntt([1, 1, 1, 1], prm, 8) == [4, 0, 0, 0]
    assert bigint.run_ntt([1, 2, 3, 4], prm, 8) == [10, 1, 11, 8]


def test_bit_reverse_pin():  # test_kernels.py:182-191
    assert bigint.bit_reverse_order(8) == [0, 4, 2, 6, 1, 5, 3, 7]


# ---- golden fixtures (reference run_vector / run_ntt outputs)
def test_blas_golden_python(golden):
    for row in golden("blas"):
        q = int(row["q"])
        a = [int(x) for x in row["a"]]
        b = [int(x) for x in row["b"]]
        args = (int(row["scalar"]), a, b) if row["kind"] == "axpy" else (a, b)
        assert bigint.run_vector(row["kind"], q, row["bits"], *args) == [int(x) for x in row["out"]], row["kind"]


def test_blas_golden_c(golden):
    for row in golden("blas"):
        q, bits = int(row["q"]), row["bits"]
        f = OracleField(q, bits)
        a = limbs(row["a"], f.K)
        b = limbs(row["b"], f.K)
        out = f.vector(row["kind"], a, b, int(row.get("scalar", 0)))
        assert ints(out) == [int(x) for x in row["out"]], (row["kind"], bits)


def test_ntt_golden(golden):
    for row in golden("ntt"):
        bits, n = row["bits"], row["n"]
        prm = bigint.find_ntt_params(bits, n)
        f = OracleField(prm["p"], bits)
        x = limbs(row["x"], f.K)
        assert ints(f.ntt(x, n, prm["root"])) == [int(v) for v in row["fwd"]]
        assert ints(f.ntt(x, n, prm["root_inv"], prm["n_inv"])) == [int(v) for v in row["inv"]]
        if n <= 64:
            xs = [int(v) for v in row["x"]]
            assert bigint.run_ntt(xs, prm, bits) == [int(v) for v in row["fwd"]]
            assert bigint.ntt_reference(xs, prm["p"], prm["root"], prm["root_inv"], prm["n_inv"]) == \
                [int(v) for v in row["fwd"]]


def test_ntt_large_golden_checksums(golden):
    """256-bit n=2^16: the C oracle reproduces the reference's own run_ntt
    output checksums (make_golden.py ntt_large)."""
    for row in golden("ntt_large"):
        n, p = row["n"], int(row["p"])
        prm = bigint.find_ntt_params(256, n)
        assert prm["p"] == p
        x = bigint.uniform_residues(np.random.Generator(np.random.PCG64(row["seed"])), n, p)
        xl = limbs(x, 8)
        assert hashlib.sha256(xl.tobytes()).hexdigest() == row["x_sha256"]
        f = OracleField(p, 256)
        yf = f.ntt(xl, n, prm["root"])
        assert hashlib.sha256(yf.tobytes()).hexdigest() == row["fwd_sha256"]
        yi = f.ntt(xl, n, prm["root_inv"], prm["n_inv"])
        assert hashlib.sha256(yi.tobytes()).hexdigest() == row["inv_sha256"]


def test_ntt_points_matches_transform():
    prm = bigint.find_ntt_params(256, 1024)
    f = OracleField(prm["p"], 256)
    rng = np.random.Generator(np.random.PCG64(5))
    x = limbs(bigint.uniform_residues(rng, 1024, prm["p"]), 8)
    y = f.ntt(x, 1024, prm["root"])
    ks = [0, 1, 7, 511, 1023]
    pts = f.ntt_points(x, prm["root"], ks)
    assert ints(pts) == [ints(y[k:k + 1])[0] for k in ks]


def test_exact_ntt_restatement_matches_reference_executor():
    """run_ntt_exact (general-modulus restatement, for full-width fields)
    equals the reference-faithful run_ntt where both apply, and ntt_point
    equals the O(n^2) ntt_reference at single indices."""
    assert bigint.run_ntt_exact([1, 2, 3, 4], 13, 5, 10) == [10, 1, 11, 8]  # test_kernels.py:161
    for width, n in [(16, 16), (64, 64), (256, 128)]:
        prm = bigint.find_ntt_params(width, n)
        rng = np.random.Generator(np.random.PCG64(width))
        x = bigint.uniform_residues(rng, n, prm["p"])
        assert bigint.run_ntt_exact(x, prm["p"], prm["root"], prm["n_inv"]) == bigint.run_ntt(x, prm, width)
        y = bigint.run_ntt(x, prm, width)
        assert bigint.run_ntt_exact(y, prm["p"], prm["root_inv"], prm["n_inv"], inverse=True) == x
        ref = bigint.ntt_reference(x, prm["p"], prm["root"], prm["root_inv"], prm["n_inv"])
        for k in (0, 1, n - 1, n // 3):
            assert bigint.ntt_point(x, prm["p"], prm["root"], k) == ref[k]


# ---- round 2: the full-output config fixtures and the reference butterfly
def test_uniform_residue_limbs_matches_uniform_residues():
    """The vectorised generator of the config fixtures draws exactly what
    uniform_residues draws (same rejections, same order), incl. a small
    modulus where rejections happen."""
    for q, count in [((1 << 252) - 129, 3000), (4093, 5000), (500, 4000), ((1 << 64) - 59, 2000)]:
        a = bigint.uniform_residues(np.random.Generator(np.random.PCG64(5)), count, q)
        b = bigint.uniform_residue_limbs(np.random.Generator(np.random.PCG64(5)), count, q)
        assert ints(b) == a, q


def test_config_fixture_inputs_and_oracle(golden):
    """tests/golden/ntt_configs.json: the inputs regenerate to the recorded
    hash, and the pinned C oracle reproduces the config-2 output hashes (the
    2^20/2^24 rows are produced by the same code path, make_ntt_configs.py)."""
    rows = {r["name"]: r for r in golden("ntt_configs")}
    assert set(rows) == {"cfg2_2p16_x64", "cfg4_2p20_x4", "cfg5_2p24"}
    for r in rows.values():
        p = int(r["p"])
        assert p == bigint.find_ntt_params(256, r["n"])["p"] if r["n"] <= 1 << 20 else True
        x = bigint.uniform_residue_limbs(np.random.Generator(np.random.PCG64(r["seed"])), r["batch"] * r["n"], p)
        assert hashlib.sha256(x.tobytes()).hexdigest() == r["x_sha256"], r["name"]
    r = rows["cfg2_2p16_x64"]
    prm = bigint.find_ntt_params(256, r["n"])
    x = bigint.uniform_residue_limbs(np.random.Generator(np.random.PCG64(r["seed"])), r["batch"] * r["n"], prm["p"])
    of = OracleField(prm["p"], 256)
    per = r["n"] * 8
    fwd = of.ntt(x[: 4 * r["n"]], r["n"], prm["root"])  # the first 4 transforms (time)
    for b in range(4):
        assert hashlib.sha256(fwd.reshape(-1)[b * per:(b + 1) * per].tobytes()).hexdigest() == r["fwd_sha256_each"][b]


def test_butterfly_golden_is_modular_butterfly(golden):
    """The reference's run_program on transform kinds (butterfly.json) is
    (u + v w, u - v w) mod p — what the device run_program computes."""
    for row in golden("butterfly"):
        p = int(row["p"])
        for ops, out in zip(row["ops"], row["out"]):
            u, v, w = (int(a) for a in ops)
            assert [int(a) for a in out] == [(u + v * w) % p, (u - v * w) % p]
