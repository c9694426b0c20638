"""Data tables users pass as INPUTS to the library (no dequantization arithmetic).

``bnb_dynamic_code2()`` is the 256-entry second-level code table QLoRA /
BitsAndBytes use for double-quantized absmax ("nested" statistics): the signed
8-bit dynamic map, ``create_dynamic_map(signed=True, max_exponent_bits=7,
total_bits=8)`` ([ext]).  It is what ``NF4Linear`` uses by
default when it double-quantizes a weight; nf4_dequantize takes whatever table
``dq_state.code2`` points to, so parity never depends on how it was built.
The test-input package (synth/) keeps its own copy; tests/test_abi.py checks the
two are identical.
"""
from __future__ import annotations

import numpy as np


def bnb_dynamic_code2() -> np.ndarray:
    vals = []
    max_exp, non_sign_bits = 7, 7
    for i in range(max_exp):
        n_frac = 2 ** (i + non_sign_bits - max_exp) + 1
        edges = np.linspace(0.1, 1.0, n_frac, dtype=np.float32)
        mids = ((edges[:-1] + edges[1:]) / np.float32(2.0)).astype(np.float64)
        scale = 10.0 ** (i - (max_exp - 1))
        vals.extend((scale * mids).tolist())
        vals.extend((-scale * mids).tolist())
    vals.extend([0.0, 1.0])
    table = np.sort(np.array(vals, dtype=np.float32))
    assert table.size == 256
    return table
