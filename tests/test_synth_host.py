"""The multi-threaded host input generator (synth/hashgen.c) draws exactly the
streams of synth/inputs.py (the reference definition of the input hash)."""
from __future__ import annotations

import numpy as np

from synth import fast
from synth import inputs as syn


def test_fast_streams_equal_numpy_definition():
    for begin, count in ((0, 1), (0, 8), (3, 5), (5, 4099), (123456789, 777), ((1 << 33) + 3, 70001)):
        assert np.array_equal(fast.packed(42, begin, count, threads=3), syn.hash_packed(42, begin, count))
        assert np.array_equal(fast.qabsmax(7, begin, count, threads=2), syn.hash_qabsmax(7, begin, count))
        assert np.array_equal(fast.absmax(9, begin, count, threads=4).view(np.uint32),
                              syn.hash_absmax(9, begin, count).view(np.uint32))
        assert np.array_equal(fast.absmax2(11, begin, count, threads=5).view(np.uint32),
                              syn.hash_absmax2(11, begin, count).view(np.uint32))


def test_fast_empty_and_thread_invariant():
    assert fast.packed(1, 10, 0).size == 0
    a = fast.packed(5, 1000, 1 << 20, threads=1)
    b = fast.packed(5, 1000, 1 << 20, threads=7)
    assert np.array_equal(a, b)
