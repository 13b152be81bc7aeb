"""Host-side behaviour of the reference-mirroring operator API
(paper_2501_07535_b200.kernels): the same validation, errors, schedules and
word conversions as reference kernels.py, checked without a GPU (no call
here launches a kernel)."""

from __future__ import annotations

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2501_07535_b200 import kernels as K
from paper_2501_07535_b200.params import NttParams, compute_barrett, find_ntt_params


def test_word_layout():  # reference test_kernels.py:36-48
    lay = K.WordLayout(24, 8)
    assert (lay.words, lay.padded_words, lay.padded_bits) == (3, 4, 32)
    assert K.WordLayout(12, 8).padded_bits == 16
    assert K.WordLayout(16, 16).padded_words == 1
    assert K.WordLayout(1024, 64).padded_words == 16
    assert K.WordLayout(384, 64).limbs == 12 and K.WordLayout(768, 32).limbs == 24
    with pytest.raises(K.InvalidKernel):
        K.WordLayout(16, 12)
    with pytest.raises(K.InvalidKernel):
        K.WordLayout(4, 8)


def test_kernel_spec_validation():  # reference test_kernels.py:51-69
    lay = K.WordLayout(16, 8)
    bp = compute_barrett(4093, 16)
    nt = find_ntt_params(16, 4)
    with pytest.raises(K.InvalidKernel):
        K.KernelSpec("frobnicate", lay, 1, bp)
    with pytest.raises(K.InvalidKernel):
        K.KernelSpec("mulmod", lay, 2, bp)
    with pytest.raises(K.InvalidKernel):
        K.KernelSpec("vadd", lay, 0, bp)
    with pytest.raises(K.InvalidKernel):
        K.KernelSpec("ntt", lay, 4, bp, None)
    with pytest.raises(K.InvalidKernel):
        K.KernelSpec("ntt", lay, 8, compute_barrett(nt.p, 16), nt)
    with pytest.raises(K.InvalidKernel):
        K.KernelSpec("addmod", lay, 1, None)
    with pytest.raises(K.InvalidKernel):
        K.KernelSpec("addmod", lay, 1, compute_barrett(13, 8))
    K.KernelSpec("ntt", lay, 4, compute_barrett(nt.p, 16), nt)


def test_make_spec_choices():  # reference test_kernels.py:72-79
    assert K.make_spec("mulmod", 16, 8).barrett.q == 4093
    ntt = K.make_spec("ntt", 16, 8, size=8)
    assert ntt.ntt.p == 4073 and ntt.barrett.q == 4073
    wm = K.make_spec("widemul", 64, 8)
    assert wm.barrett is None and wm.ntt is None


def test_generate_kernel_attributes():
    prog = K.generate_kernel(K.make_spec("vmul", 256, 64, size=1 << 16))
    a = prog.attributes
    assert prog.name == "vmul65536_256w64"
    assert a["n"] == 1 << 16 and a["vector_args"] == [True, True] and a["limbs"] == 8
    ax = K.generate_kernel(K.make_spec("axpy", 128, 64, size=8))
    assert ax.attributes["vector_args"] == [False, True, True]
    rt = K.generate_kernel(K.make_spec("mulmod", 16, 8), params_mode="runtime")
    assert rt.attributes["arg_names"] == ["a", "b", "q", "mu"]  # reference test_kernels.py:103-107
    nt = K.generate_kernel(K.make_spec("intt", 16, 8, size=8))
    assert nt.attributes["direction"] == "inverse" and nt.name == "intt8_16w8"
    assert [int(x) for x in nt.attributes["twiddles"]] == K.twiddle_table(find_ntt_params(16, 8), inverse=True)
    with pytest.raises(K.InvalidKernel):
        K.generate_kernel(K.make_spec("vadd", 16, 8, size=4), params_mode="wat")
    wm = K.generate_kernel(K.make_spec("widemul", 64, 8))  # reference build_wide_mul kernels.py:314-329
    assert wm.name == "widemul_64w8" and wm.attributes["ret_names"] == ["c"]
    with pytest.raises(K.InvalidKernel):
        wm.modulus


def test_run_vector_validation_before_launch():  # reference test_kernels.py:137-144
    vadd = K.generate_kernel(K.make_spec("vadd", 16, 8, size=4))
    with pytest.raises(ValueError):
        K.run_vector(vadd, [1, 2, 3], [1, 2, 3, 4])
    with pytest.raises(TypeError):
        K.run_vector(vadd, [1, 2, 3, 4])
    ntt = K.generate_kernel(K.make_spec("ntt", 8, 8, size=4))
    with pytest.raises(ValueError):  # reference test_kernels.py:278-281
        K.run_ntt(ntt, [1, 2, 3])
    add = K.generate_kernel(K.make_spec("addmod", 16, 8))
    with pytest.raises(TypeError):  # reference test_kernels.py:272-275
        K.run_program(add, 1, 2, 3)


def test_twiddle_table_pinned():  # reference test_kernels.py:147-153
    assert K.twiddle_table(find_ntt_params(8, 4)) == [1, 5]
    p17 = NttParams(n=8, p=17, root=2, root_inv=9, n_inv=15)
    assert K.twiddle_table(p17) == [1, 2, 4, 8]
    assert K.twiddle_table(p17, inverse=True) == [1, 9, 13, 15]


def test_bit_reverse_order():  # reference test_kernels.py:182-191
    assert K.bit_reverse_order(1) == [0]
    assert K.bit_reverse_order(2) == [0, 1]
    assert K.bit_reverse_order(8) == [0, 4, 2, 6, 1, 5, 3, 7]
    for n in (4, 16, 64):
        rev = K.bit_reverse_order(n)
        assert sorted(rev) == list(range(n)) and all(rev[rev[i]] == i for i in range(n))
    with pytest.raises(K.InvalidKernel):
        K.bit_reverse_order(3)


@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64])
def test_butterfly_schedule_shape(n):  # reference test_kernels.py:194-204
    sched = K.butterfly_schedule(n)
    assert len(sched) == (n // 2) * (n.bit_length() - 1)
    per = n // 2
    for s in range(n.bit_length() - 1):
        stage = sched[s * per:(s + 1) * per]
        assert sorted(i for t, b, _ in stage for i in (t, b)) == list(range(n))
        assert all(e < n // 2 for _, _, e in stage)
    with pytest.raises(K.InvalidKernel):
        K.butterfly_schedule(6)


def test_words_roundtrip():  # reference test_kernels.py:214-217
    assert K.to_words(0x0102, 2, 8) == [1, 2]
    assert K.from_words([1, 2], 8) == 0x0102
    assert K.to_words(5, 4, 8) == [0, 0, 0, 5]


@given(st.integers(0, (1 << 64) - 1), st.sampled_from([8, 16, 32, 64]))
@settings(max_examples=50)
def test_words_roundtrip_property(value, width):  # reference test_kernels.py:220-224
    count = 64 // width
    assert K.from_words(K.to_words(value, count, width), width) == value


def test_limb_conversion_roundtrip():
    from paper_2501_07535_b200.device import ints_to_limbs, limbs_to_ints
    vals = [0, 1, (1 << 252) - 129, 12345678901234567890]
    arr = ints_to_limbs(vals, 8)
    assert arr.shape == (4, 8) and arr[1, 0] == 1 and arr[1, 1:].sum() == 0
    assert limbs_to_ints(arr) == vals
    with pytest.raises(ValueError):
        ints_to_limbs([1 << 256], 8)
