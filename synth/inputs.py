"""Seeded input generators (no method arithmetic; see synth/__init__.py).

Two families of inputs:

1. *Realistic* (small sizes, tests):  ``gaussian_weights`` draws W ~ N(0, std^2)
   fp32 with numpy's counter-based Philox generator -- the paper's premise that
   LLM weights are normally distributed.  Tests quantize them with the
   oracle quantizer to obtain packed codes + absmax (+ double-quant state).

2. *Counter-based hash* (any size, full-size GPU parity):  every packed byte,
   absmax, qabsmax byte and absmax2 value is a pure function of
   (seed, stream, index) through the SplitMix64 finaliser below.  The CUDA side
   implements the same function (csrc/synth_gen.cu), so full-size inputs are
   generated on the device while the oracle regenerates any sampled block on
   the host.  Value ranges mimic NF4-quantized N(0, 0.02^2) weights: codes are
   near-uniform over 0..15 (NF4 levels are equal-probability quantiles), block
   absmax in [2^-5, 2^-4) (max |w| of 64 draws is ~2.4 sigma ~ 0.048), second-
   level scales in [2^-6, 2^-5), offset in [0.046875, 0.0625).  Floats are built
   directly from bits (no floating-point arithmetic), so both sides agree
   exactly.
"""
from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# Counter-based hash (SplitMix64 finaliser of a Weyl-style key)
# ---------------------------------------------------------------------------
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
STREAM_MUL = np.uint64(0xD1B54A32D192ED03)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

STREAM_CODES = 1
STREAM_ABSMAX = 2
STREAM_QABSMAX = 3
STREAM_ABSMAX2 = 4
STREAM_OFFSET = 5


def hash64(seed: int, stream: int, idx) -> np.ndarray:
    """z = splitmix64_mix(seed*GOLDEN + stream*STREAM_MUL + idx), all mod 2^64."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        key = (np.full(idx.shape, seed, np.uint64) * GOLDEN
               + np.full(idx.shape, stream, np.uint64) * STREAM_MUL + idx)
        z = key
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        z = z ^ (z >> np.uint64(31))
    return z


def hash_bytes(seed: int, stream: int, byte_begin: int, count: int) -> np.ndarray:
    """Bytes [byte_begin, byte_begin+count) of the stream: byte j is byte (j % 8)
    (little-endian) of hash64(seed, stream, j // 8)."""
    if count <= 0:
        return np.zeros(0, np.uint8)
    w0 = byte_begin // 8
    w1 = (byte_begin + count + 7) // 8
    words = hash64(seed, stream, np.arange(w0, w1, dtype=np.uint64))
    raw = words.astype("<u8").view(np.uint8)
    off = byte_begin - 8 * w0
    return raw[off:off + count].copy()


def _float_from_bits(seed, stream, idx, base_bits: int, mant_bits: int) -> np.ndarray:
    z = hash64(seed, stream, idx)
    bits = (np.uint64(base_bits) | (z & np.uint64((1 << mant_bits) - 1))).astype(np.uint32)
    return bits.view(np.float32)


def hash_packed(seed: int, byte_begin: int, count: int) -> np.ndarray:
    return hash_bytes(seed, STREAM_CODES, byte_begin, count)


def hash_absmax(seed: int, block_begin: int, count: int) -> np.ndarray:
    """fp32 absmax in [2^-5, 2^-4): exponent 122, 23 random fraction bits."""
    idx = np.arange(block_begin, block_begin + count, dtype=np.uint64)
    return _float_from_bits(seed, STREAM_ABSMAX, idx, 0x3D000000, 23)


def hash_qabsmax(seed: int, block_begin: int, count: int) -> np.ndarray:
    return hash_bytes(seed, STREAM_QABSMAX, block_begin, count)


def hash_absmax2(seed: int, group_begin: int, count: int) -> np.ndarray:
    """fp32 second-level scales in [2^-6, 2^-5): exponent 121."""
    idx = np.arange(group_begin, group_begin + count, dtype=np.uint64)
    return _float_from_bits(seed, STREAM_ABSMAX2, idx, 0x3C800000, 23)


def hash_offset(seed: int) -> np.float32:
    """DQ offset in [0.046875, 0.0625): exponent 122, top fraction bit set."""
    return _float_from_bits(seed, STREAM_OFFSET, np.zeros(1, np.uint64), 0x3D400000, 22)[0]


# ---------------------------------------------------------------------------
# Realistic small inputs
# ---------------------------------------------------------------------------
def gaussian_weights(n: int, seed: int, std: float = 0.02) -> np.ndarray:
    """W ~ N(0, std^2) as fp32, numpy Philox stream keyed by ``seed``."""
    rng = np.random.Generator(np.random.Philox(seed))
    return (rng.standard_normal(n, dtype=np.float32) * np.float32(std)).astype(np.float32)


def dynamic_map_code2() -> np.ndarray:
    """The 256-entry signed 8-bit dynamic code used by QLoRA/BNB double quantization
    for the second-level absmax codes (create_dynamic_map(signed=True,
    max_exponent_bits=7, total_bits=8); [ext]).  It is an
    INPUT to dequantization (dq_state.code2): parity never depends on how it was
    built.  Built here with float32 linspace like the original."""
    data = []
    max_exp, non_sign_bits = 7, 7
    for i in range(max_exp):
        fraction_items = 2 ** (i + non_sign_bits - max_exp) + 1
        bnd = np.linspace(0.1, 1.0, fraction_items, dtype=np.float32)
        means = (bnd[:-1] + bnd[1:]) / np.float32(2.0)
        scale = 10.0 ** (-(max_exp - 1) + i)
        data += (scale * means.astype(np.float64)).tolist()
        data += (-scale * means.astype(np.float64)).tolist()
    data.append(0.0)
    data.append(1.0)
    assert len(data) == 256
    return np.sort(np.array(data, dtype=np.float32))


def bnb_fp4_codebook() -> np.ndarray:
    """BitsAndBytes' 16-entry FP4 table ([ext]: bnb get_4bit_type('fp4'): sign, 2-bit
    exponent, 1-bit mantissa values {0, 0.0625, 8, 12, 4, 6, 2, 3} and negatives,
    divided by their max).  An INPUT to nf4_dequantize_ex."""
    data = np.array([0, 0.0625, 8.0, 12.0, 4.0, 6.0, 2.0, 3.0,
                     -0.0, -0.0625, -8.0, -12.0, -4.0, -6.0, -2.0, -3.0], np.float32)
    return (data / np.float32(12.0)).astype(np.float32)


def random_codes(n_bytes: int, seed: int) -> np.ndarray:
    rng = np.random.Generator(np.random.Philox(seed))
    return rng.integers(0, 256, n_bytes, dtype=np.uint8)
