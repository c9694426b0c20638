"""Independent numpy expressions used only to PIN the C oracle (tests only).

Different route from oracle/oracle.c: numpy fancy indexing instead of a scalar
loop, numpy's float32 multiply, and the *library* fp32->fp16 / fp32->bf16
conversions (torch CPU / numpy / ml_dtypes) instead of the oracle's
hand-written integer round-to-nearest-even.  Never used against the GPU path.
"""
from __future__ import annotations

import ml_dtypes
import numpy as np

# QLoRA NF4 table as decimals (S:40-43 for entries 0,1,7,15)
NF4_DECIMAL = np.array([
    -1.0, -0.6961928009986877, -0.5250730514526367, -0.39491748809814453,
    -0.28444138169288635, -0.18477343022823334, -0.09105003625154495, 0.0,
    0.07958029955625534, 0.16093020141124725, 0.24611230194568634, 0.33791524171829224,
    0.44070982933044434, 0.5626170039176941, 0.7229568362236023, 1.0], dtype=np.float64)


def to16(p: np.ndarray, dtype: str) -> np.ndarray:
    p = np.asarray(p, np.float32)
    if dtype == "f16":
        with np.errstate(over="ignore"):
            return p.astype(np.float16).view(np.uint16)
    return p.astype(ml_dtypes.bfloat16).view(np.uint16)


def dequant_np(packed, n, bs, dtype, absmax=None, qabsmax=None, code2=None, absmax2=None,
               offset=0.0, bs2=256, codebook=None):
    cb = NF4_DECIMAL.astype(np.float32) if codebook is None else np.asarray(codebook, np.float32)
    k = np.arange(n, dtype=np.int64)
    byte = packed[k >> 1]
    idx = np.where(k % 2 == 0, byte >> 4, byte & 0x0F)
    b = k // bs
    if absmax is not None:
        a = absmax[b]
    else:
        t = (code2[qabsmax[b]] * absmax2[b // bs2]).astype(np.float32)
        a = (t + np.float32(offset)).astype(np.float32)
    p = (cb[idx] * a).astype(np.float32)
    if dtype == "f32":
        return p.view(np.uint32)
    return to16(p, dtype)


def same_bits(a16: np.ndarray, b16: np.ndarray, dtype: str) -> np.ndarray:
    """Bitwise equality, except any-NaN == any-NaN (NaN payloads differ, reading R9)."""
    a16 = np.asarray(a16, np.uint16)
    b16 = np.asarray(b16, np.uint16)
    if dtype == "f16":
        na = ((a16 & 0x7C00) == 0x7C00) & ((a16 & 0x03FF) != 0)
        nb = ((b16 & 0x7C00) == 0x7C00) & ((b16 & 0x03FF) != 0)
    else:
        na = ((a16 & 0x7F80) == 0x7F80) & ((a16 & 0x007F) != 0)
        nb = ((b16 & 0x7F80) == 0x7F80) & ((b16 & 0x007F) != 0)
    return np.where(na | nb, na & nb, a16 == b16)
