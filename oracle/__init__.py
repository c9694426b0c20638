"""CPU oracle for blockwise NF4 dequantization (arxiv 2604.02556).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product package ``paper_2604_02556_b200`` never imports it and
shares no code with it.

The arithmetic lives in ``oracle.c`` (plain scalar C, fp32 IEEE, no FMA
contraction, no FTZ/DAZ); this module only compiles it with gcc and marshals
numpy arrays through ctypes.  Every function is pinned by
``tests/test_oracle_pins.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OUT_F16 = 0
OUT_BF16 = 1
OUT_F32 = 2

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.run(["gcc", *CFLAGS, "-o", tmp, _SRC], check=True)
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i64, i32, f32 = ctypes.c_int64, ctypes.c_int32, ctypes.c_float
            lib.oracle_nf4_codebook.argtypes = [P]
            lib.oracle_nf4_thresholds.argtypes = [P]
            lib.oracle_f32_to_f16.argtypes = [ctypes.c_uint32]
            lib.oracle_f32_to_f16.restype = ctypes.c_uint16
            lib.oracle_f32_to_bf16.argtypes = [ctypes.c_uint32]
            lib.oracle_f32_to_bf16.restype = ctypes.c_uint16
            lib.oracle_f32_to_f16_bulk.argtypes = [P, i64, P]
            lib.oracle_f32_to_bf16_bulk.argtypes = [P, i64, P]
            lib.oracle_dequantize.argtypes = [P, P, P, P, P, f32, i32, i64, i32, i32, i64, i64, P]
            lib.oracle_dequantize.restype = ctypes.c_int
            lib.oracle_dequantize_ex.argtypes = [P, P, P, P, P, f32, i32, i64, i32, P, i32, i64, i64, P]
            lib.oracle_dequantize_ex.restype = ctypes.c_int
            lib.oracle_quantize.argtypes = [P, i64, i32, P, P]
            lib.oracle_quantize.restype = ctypes.c_int
            lib.oracle_double_quantize.argtypes = [P, i64, f32, P, i32, P, P]
            lib.oracle_double_quantize.restype = ctypes.c_int
            _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def _c(a, dtype):
    if a is None:
        return None
    a = np.ascontiguousarray(a)
    if a.dtype != dtype:
        raise TypeError(f"expected {dtype}, got {a.dtype}")
    return a


def codebook() -> np.ndarray:
    out = np.zeros(16, np.float32)
    _load().oracle_nf4_codebook(_ptr(out))
    return out


def thresholds() -> np.ndarray:
    out = np.zeros(15, np.float32)
    _load().oracle_nf4_thresholds(_ptr(out))
    return out


def f32_to_f16_bits(x_bits: np.ndarray) -> np.ndarray:
    x = _c(x_bits, np.uint32)
    out = np.empty(x.shape, np.uint16)
    _load().oracle_f32_to_f16_bulk(_ptr(x), x.size, _ptr(out))
    return out


def f32_to_bf16_bits(x_bits: np.ndarray) -> np.ndarray:
    x = _c(x_bits, np.uint32)
    out = np.empty(x.shape, np.uint16)
    _load().oracle_f32_to_bf16_bulk(_ptr(x), x.size, _ptr(out))
    return out


def dequantize(packed, n, blocksize, out_dtype, absmax=None, qabsmax=None, code2=None,
               absmax2=None, offset=0.0, blocksize2=256, k_begin=0, k_end=None,
               threads: int = 1, codebook=None) -> np.ndarray:
    """Oracle dequantization; returns the raw output words (uint16 for fp16/bf16,
    uint32 fp32 bits for OUT_F32).  ``codebook``: optional 16-entry fp32 table
    (default NF4).

    Exactly one of ``absmax`` (fp32 mode) or ``qabsmax``+``code2``+``absmax2``
    (double-quant mode) must be given.  ``threads`` > 1 splits [k_begin, k_end)
    into contiguous ranges run concurrently (ctypes releases the GIL); the
    arithmetic is the same scalar loop.
    """
    lib = _load()
    packed = _c(packed, np.uint8)
    absmax = _c(absmax, np.float32)
    qabsmax = _c(qabsmax, np.uint8)
    code2 = _c(code2, np.float32)
    absmax2 = _c(absmax2, np.float32)
    cb = _c(codebook, np.float32)
    if cb is not None and cb.size != 16:
        raise ValueError("codebook must have 16 entries")
    if k_end is None:
        k_end = n
    m = k_end - k_begin
    wsz = 4 if out_dtype == OUT_F32 else 2
    out = np.empty(max(m, 0), np.uint32 if wsz == 4 else np.uint16)

    def run(a, b):
        rc = lib.oracle_dequantize_ex(_ptr(packed), _ptr(absmax), _ptr(qabsmax), _ptr(code2),
                                      _ptr(absmax2), float(offset), int(blocksize2), int(n),
                                      int(blocksize), _ptr(cb), int(out_dtype), int(a), int(b),
                                      out.ctypes.data + wsz * (a - k_begin))
        if rc != 0:
            raise ValueError(f"oracle_dequantize rejected its arguments (rc={rc})")

    if threads <= 1 or m < 1 << 16:
        run(k_begin, k_end)
    else:
        step = -(-m // threads)
        step = -(-step // 2) * 2
        ranges = [(k_begin + i * step, min(k_end, k_begin + (i + 1) * step)) for i in range(threads)]
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda r: run(*r), [r for r in ranges if r[0] < r[1]]))
    return out


def quantize(x: np.ndarray, blocksize: int):
    """Oracle NF4 quantizer (input generator): returns (packed uint8, absmax fp32)."""
    x = _c(x, np.float32)
    n = x.size
    packed = np.zeros((n + 1) // 2, np.uint8)
    absmax = np.zeros((n + blocksize - 1) // blocksize, np.float32)
    rc = _load().oracle_quantize(_ptr(x), n, int(blocksize), _ptr(packed), _ptr(absmax))
    if rc != 0:
        raise ValueError("oracle_quantize rejected its arguments")
    return packed, absmax


def double_quantize(absmax: np.ndarray, offset: float, code2: np.ndarray, blocksize2: int = 256):
    """Oracle second-level quantizer (input generator): returns (qabsmax uint8, absmax2 fp32)."""
    absmax = _c(absmax, np.float32)
    code2 = _c(code2, np.float32)
    nb = absmax.size
    q = np.zeros(nb, np.uint8)
    a2 = np.zeros((nb + blocksize2 - 1) // blocksize2, np.float32)
    rc = _load().oracle_double_quantize(_ptr(absmax), nb, float(np.float32(offset)), _ptr(code2),
                                        int(blocksize2), _ptr(q), _ptr(a2))
    if rc != 0:
        raise ValueError("oracle_double_quantize rejected its arguments")
    return q, a2


def gemm_reference(x16: np.ndarray, x_dtype: int, packed, N: int, K: int, blocksize: int, **scale_kw):
    """Reference for the fused GEMM: W = this oracle's dequantization
    of the NF4 weight [N, K] into x's 16-bit type (bit-exact hot-path values), then
    Y = X . W^T with numpy in fp64 (a library matmul as one step).  Returns
    (Y fp64 [M, N], S fp64 [M, N] = sum_k |x_mk w_nk|) -- S bounds the fp32
    accumulation error of any summation order: |Y_gpu - Y| <= K * 2^-23 * S.
    Pinned (tests/test_oracle_pins.py): one-hot / all-ones X against the rounded
    codebook (closed form), exact linearity for integer X, S >= |Y| and S == Y for
    non-negative operands."""
    import ml_dtypes
    w16 = dequantize(packed, N * K, blocksize, x_dtype, threads=8, **scale_kw)
    np16 = np.float16 if x_dtype == OUT_F16 else ml_dtypes.bfloat16
    w = w16.view(np16).astype(np.float64).reshape(N, K)
    x = np.asarray(x16, np.uint16).view(np16).astype(np.float64).reshape(-1, K)
    return x @ w.T, np.abs(x) @ np.abs(w).T
