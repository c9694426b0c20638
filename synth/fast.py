"""Multi-threaded host fill of the counter-based input streams (synth/hashgen.c).

Same values as ``synth.inputs.hash_packed`` / ``hash_absmax`` / ``hash_qabsmax`` /
``hash_absmax2`` (pinned by tests/test_synth_host.py), at GB/s instead of the
numpy version's ~0.1 GB/s, so the full-size parity tests can regenerate every
input of a 68 G-element workload on the host.  Input generation only -- none
of the method's arithmetic.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import inputs as _inp

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hashgen.c")
_LIB = os.path.join(_HERE, "libsynth.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", tmp, _SRC], check=True)
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            u64, i64, u32, P = ctypes.c_uint64, ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p
            lib.synth_fill_bytes.argtypes = [u64, u64, i64, i64, P]
            lib.synth_fill_f32.argtypes = [u64, u64, i64, i64, u32, u32, P]
            if not lib.synth_little_endian():
                raise RuntimeError("synth/hashgen.c assumes a little-endian host")
            _lib = lib
    return _lib


def _threads(threads):
    return threads or len(os.sched_getaffinity(0))


def _split(count, threads, align):
    step = -(-count // threads)
    step = -(-step // align) * align
    return [(i, min(count, i + step)) for i in range(0, count, step)] if count > 0 else []


def fill_bytes(seed: int, stream: int, begin: int, count: int, threads=None, out=None) -> np.ndarray:
    lib = _load()
    out = np.empty(count, np.uint8) if out is None else out
    base = out.ctypes.data

    def run(r):
        a, b = r
        lib.synth_fill_bytes(seed, stream, begin + a, b - a, base + a)

    with ThreadPoolExecutor(_threads(threads)) as ex:
        list(ex.map(run, _split(count, _threads(threads), 1 << 16)))
    return out


def fill_f32(seed: int, stream: int, begin: int, count: int, base_bits: int, mant_bits: int,
             threads=None) -> np.ndarray:
    lib = _load()
    out = np.empty(count, np.uint32)
    ptr = out.ctypes.data
    mask = (1 << mant_bits) - 1

    def run(r):
        a, b = r
        lib.synth_fill_f32(seed, stream, begin + a, b - a, base_bits, mask, ptr + 4 * a)

    with ThreadPoolExecutor(_threads(threads)) as ex:
        list(ex.map(run, _split(count, _threads(threads), 1 << 14)))
    return out.view(np.float32)


# the same streams and bit layouts as synth.inputs
def packed(seed, byte_begin, count, threads=None):
    return fill_bytes(seed, _inp.STREAM_CODES, byte_begin, count, threads)


def qabsmax(seed, block_begin, count, threads=None):
    return fill_bytes(seed, _inp.STREAM_QABSMAX, block_begin, count, threads)


def absmax(seed, block_begin, count, threads=None):
    return fill_f32(seed, _inp.STREAM_ABSMAX, block_begin, count, 0x3D000000, 23, threads)


def absmax2(seed, group_begin, count, threads=None):
    return fill_f32(seed, _inp.STREAM_ABSMAX2, group_begin, count, 0x3C800000, 23, threads)
