"""The reference's named kernel builders (build_scalar / build_vector /
build_ntt / build_wide_mul, reference kernels.py:184-329) on the device.

CPU tests check the validation and the Program-shaped metadata (names,
argument lists) without launching anything; ``gpu`` tests run the reference's
own pinned values (reference tests/test_kernels.py:82-176) through
run_program / run_vector / run_ntt, plus random cases against Python ints."""

from __future__ import annotations

import random

import pytest

from paper_2501_07535_b200 import kernels as K
from paper_2501_07535_b200.params import NttParams, compute_barrett, find_ntt_params

L13 = K.WordLayout(13, 8)
Q500 = compute_barrett(500, 13)


# ------------------------------------------------------------------ CPU
def test_builders_validate_like_the_reference():  # reference test_kernels.py:137-145, 171-176
    with pytest.raises(K.InvalidKernel):
        K.build_vector("addmod", L13, 4, Q500)
    with pytest.raises(K.InvalidKernel):
        K.build_vector("vadd", L13, 0, Q500)
    with pytest.raises(K.InvalidKernel):
        K.build_vector("vadd", L13, 4, Q500, params_mode="jit")
    with pytest.raises(K.InvalidKernel):
        K.build_scalar("vadd", L13, Q500)
    with pytest.raises(K.InvalidKernel):
        K.build_scalar("addmod", L13, Q500, params_mode="jit")
    with pytest.raises(K.InvalidKernel):
        K.build_ntt("ntt", K.WordLayout(16, 8), NttParams(n=3, p=13, root=3, root_inv=9, n_inv=9))
    with pytest.raises(K.InvalidKernel):
        K.build_ntt("addmod", K.WordLayout(16, 8), find_ntt_params(16, 4))


def test_builder_metadata():  # names and argument lists of reference kernels.py:201-212, 244-256, 294-311
    s = K.build_scalar("mulmod", K.WordLayout(16, 8), compute_barrett(4093, 16), params_mode="runtime")
    assert s.name == "mulmod_16w8"
    assert s.attributes["arg_names"] == ["a", "b", "q", "mu"]
    assert K.build_scalar("addmod", L13, Q500, params_mode="runtime").attributes["arg_names"] == ["a", "b", "q"]
    v = K.build_vector("axpy", L13, 3, Q500)
    assert v.name == "axpy3_13w8" and v.attributes["n"] == 3
    assert v.attributes["arg_names"] == ["a", "x", "y"] and v.attributes["vector_args"] == [False, True, True]
    prm = find_ntt_params(8, 4)
    t = K.build_ntt("intt", K.WordLayout(8, 8), prm)
    assert t.name == "intt4_8w8" and t.attributes["direction"] == "inverse"
    assert t.attributes["q"] == str(prm.p) and t.attributes["twiddles"] == [str(x) for x in K.twiddle_table(prm, True)]
    w = K.build_wide_mul(K.WordLayout(16, 8))
    assert w.name == "widemul_16w8" and w.attributes["ret_names"] == ["c"]
    # build_program dispatches to the same handles (reference kernels.py:332-340)
    assert K.build_program(K.make_spec("vmul", 256, 64, size=8)).name == "vmul8_256w64"


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_build_scalar_pinned_values(cuda):  # reference test_kernels.py:82-91, 103-110
    assert K.run_program(K.build_scalar("addmod", L13, Q500), 300, 400) == 200
    assert K.run_program(K.build_scalar("submod", L13, Q500), 100, 300) == 300
    mm = K.build_scalar("mulmod", K.WordLayout(16, 8), compute_barrett(4093, 16))
    assert K.run_program(mm, 3000, 2000) == 3755
    rt = K.build_scalar("mulmod", K.WordLayout(16, 8), compute_barrett(4093, 16), params_mode="runtime")
    assert K.run_program(rt, 3000, 2000) == 3755


@pytest.mark.gpu
def test_build_scalar_matches_python_ints(cuda):  # reference test_kernels.py:94-100
    r = random.Random(5)
    progs = {k: K.build_scalar(k, L13, Q500) for k in K.SCALAR_KINDS}
    for _ in range(20):
        a, b = r.randrange(500), r.randrange(500)
        assert K.run_program(progs["addmod"], a, b) == (a + b) % 500
        assert K.run_program(progs["submod"], a, b) == (a - b) % 500
        assert K.run_program(progs["mulmod"], a, b) == a * b % 500


@pytest.mark.gpu
def test_build_vector_pinned_values(cuda):  # reference test_kernels.py:113-121, 137-140
    vadd = K.build_vector("vadd", L13, 4, Q500)
    assert K.run_vector(vadd, [300, 499, 0, 250], [400, 1, 0, 250]) == [200, 0, 0, 0]
    assert K.run_vector(K.build_vector("axpy", L13, 3, Q500), 0, [5, 6, 7], [9, 8, 7]) == [9, 8, 7]
    assert K.run_vector(K.build_vector("vmul", L13, 3, Q500), [1, 1, 1], [123, 456, 499]) == [123, 456, 499]
    with pytest.raises(ValueError):
        K.run_vector(vadd, [1, 2, 3], [1, 2, 3, 4])


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [13, 128, 256, 384, 768])
def test_build_vector_matches_python_ints(cuda, bits):  # reference test_kernels.py:124-134
    q = 500 if bits == 13 else find_ntt_params(bits, 1).p
    bp = compute_barrett(q, bits)
    lay = K.WordLayout(bits, 8 if bits == 13 else 64)
    r = random.Random(bits)
    n = 64
    x = [r.randrange(q) for _ in range(n)]
    y = [r.randrange(q) for _ in range(n)]
    a = r.randrange(q)
    assert K.run_vector(K.build_vector("vsub", lay, n, bp), x, y) == [(u - v) % q for u, v in zip(x, y)]
    assert K.run_vector(K.build_vector("vmul", lay, n, bp), x, y) == [u * v % q for u, v in zip(x, y)]
    assert K.run_vector(K.build_vector("axpy", lay, n, bp), a, x, y) == [(a * u + v) % q for u, v in zip(x, y)]


@pytest.mark.gpu
def test_build_ntt_pinned_transforms(cuda):  # reference test_kernels.py:156-168
    params = find_ntt_params(8, 4)
    fwd = K.build_ntt("ntt", K.WordLayout(8, 8), params)
    inv = K.build_ntt("intt", K.WordLayout(8, 8), params)
    assert K.run_ntt(fwd, [1, 0, 0, 0]) == [1, 1, 1, 1]
    assert K.run_ntt(fwd, [1, 1, 1, 1]) == [4, 0, 0, 0]
    assert K.run_ntt(fwd, [1, 2, 3, 4]) == [10, 1, 11, 8]
    r = random.Random(3)
    for _ in range(10):
        vec = [r.randrange(13) for _ in range(4)]
        assert K.run_ntt(inv, K.run_ntt(fwd, vec)) == vec
    # one butterfly through run_program: (u + v w, u - v w) mod p
    assert K.run_program(fwd, 3, 4, 5) == ((3 + 20) % params.p, (3 - 20) % params.p)


@pytest.mark.gpu
def test_build_wide_mul(cuda):  # reference kernels.py:314-329
    w = K.build_wide_mul(K.WordLayout(256, 64))
    r = random.Random(9)
    xs = [r.getrandbits(256) for _ in range(16)]
    ys = [r.getrandbits(256) for _ in range(16)]
    assert K.run_vector(w, xs, ys) == [a * b for a, b in zip(xs, ys)]
    assert K.run_program(w, (1 << 256) - 1, (1 << 256) - 1) == ((1 << 256) - 1) ** 2
