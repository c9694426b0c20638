"""Seeded synthetic inputs and workload shapes shared by tests, smoke() and bench.py.

This package holds NONE of the method's arithmetic (no codebook lookup, no scale
decode, no product, no rounding to 16 bits).  It only draws inputs:

* ``inputs``    -- Gaussian weights (numpy Philox), the 256-entry second-level
                   code table, and a counter-based hash generator for packed
                   codes / absmax / double-quant state at any index;
* ``workloads`` -- the linear-layer shapes of the paper's three models and the
                   five BASELINE.json configurations.

Both the oracle side (numpy) and the CUDA side (csrc/synth_gen.cu implements the
same counter-based hash) generate identical inputs from the same seed, so no
oracle input ever comes from the CUDA path.
"""
from . import inputs, workloads  # noqa: F401
