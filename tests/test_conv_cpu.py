"""Python int <-> limb marshalling of the drop-in calls (reference
to_words/from_words, kernels.py:418-428): the C extension (_wmconv) and the
pure-Python path agree bit for bit and reject the same inputs.  CPU only."""

from __future__ import annotations

import random

import numpy as np
import pytest


def test_int_limb_conversion_edges():
    from paper_2501_07535_b200 import device as dev
    rng = random.Random(3)
    for limbs in (1, 2, 8, 24, 32):
        vals = [0, 1, (1 << (32 * limbs)) - 1] + [rng.getrandbits(32 * limbs) for _ in range(1000)]
        arr = dev.ints_to_limbs(vals, limbs)
        assert arr.dtype == np.uint32 and arr.shape == (len(vals), limbs)
        assert dev.limbs_to_ints(arr) == vals
        want = np.frombuffer(b"".join(v.to_bytes(4 * limbs, "little") for v in vals), dtype="<u4")
        assert np.array_equal(arr.reshape(-1), want)
        with pytest.raises(ValueError):
            dev.ints_to_limbs([1 << (32 * limbs)], limbs)
        with pytest.raises(ValueError):
            dev.ints_to_limbs([-1], limbs)


def test_extension_and_python_paths_agree():
    from paper_2501_07535_b200 import device as dev
    if dev._wmconv is None:
        pytest.skip("_wmconv not built on this host")
    rng = random.Random(11)
    vals = [rng.getrandbits(251) for _ in range(5000)]
    a = dev.ints_to_limbs(vals, 8)
    ext = dev._wmconv
    try:
        dev._wmconv = None
        b = dev.ints_to_limbs(vals, 8)
        back = dev.limbs_to_ints(a)
    finally:
        dev._wmconv = ext
    assert np.array_equal(a, b) and back == vals
    assert dev.ints_to_limbs(iter(vals[:10]), 8).shape == (10, 8)  # any iterable
