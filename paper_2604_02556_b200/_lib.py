"""ctypes loader for libnf4.so (the C-ABI declared in include/nf4.h, include/nf4_tools.h).

Argument marshalling only: every step of the path runs in the library's CUDA
kernels.  If the library is missing this raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libnf4.so")


def lib_path() -> str:
    """The in-tree library; NF4_LIB (diagnostics, tools/) may name an alternative
    build of the same sources, read when the library is first loaded."""
    return os.path.abspath(os.environ["NF4_LIB"]) if os.environ.get("NF4_LIB") else LIB_PATH

NF4_OK = 0
NF4_F16, NF4_BF16, NF4_F32 = 0, 1, 2
NF4_SYNTH_CODES, NF4_SYNTH_ABSMAX, NF4_SYNTH_QABSMAX, NF4_SYNTH_ABSMAX2 = 1, 2, 3, 4
NF4_MAX_BATCH = 128

# Every symbol the public headers declare (tests/test_abi.py checks the
# headers and the .so against this list).
EXPORTS = [
    "nf4_dequantize", "nf4_dequantize_batched", "nf4_dequantize_host", "nf4_host_workspace_bytes",
    "nf4_quantize", "nf4_double_quantize", "nf4_codebook", "nf4_status_string", "nf4_last_launch_count",
    "nf4_synth_fill", "nf4_sol_stream", "nf4_set_max_ctas", "nf4_dequant_grid", "nf4_dequant_tile_elems",
    "nf4_kernel_variant_count", "nf4_kernel_variant_name", "nf4_set_kernel_variant", "nf4_get_kernel_variant",
    "nf4_dequantize_ex", "nf4_dequantize_batched_ex", "nf4_codebook_fp4",
    "nf4_gemm", "nf4_gemm_default_splits", "nf4_gemm_workspace_bytes", "nf4_dequantize_host_batched",
    "nf4_gemm_grouped", "nf4_gemm_grouped_workspace_bytes",
    "nf4_gemm_multi", "nf4_gemm_multi_workspace_bytes", "nf4_gemm_set_early_weight_reads",
    "nf4_set_early_input_reads",
]


class DQState(ctypes.Structure):
    """nf4_dq_state"""
    _fields_ = [("qabsmax", ctypes.c_void_p), ("code2", ctypes.c_void_p), ("absmax2", ctypes.c_void_p),
                ("offset", ctypes.c_float), ("blocksize2", ctypes.c_int32)]


class GemmWeight(ctypes.Structure):
    """nf4_gemm_weight"""
    _fields_ = [("packed", ctypes.c_void_p), ("absmax", ctypes.c_void_p), ("dq", DQState),
                ("N", ctypes.c_int32), ("y", ctypes.c_void_p)]


NF4_GEMM_MAX_GROUP = 4
NF4_GEMM_MAX_MULTI = 64


class GemmProblem(ctypes.Structure):
    """nf4_gemm_problem"""
    _fields_ = [("x", ctypes.c_void_p), ("K", ctypes.c_int32), ("packed", ctypes.c_void_p),
                ("absmax", ctypes.c_void_p), ("dq", DQState), ("N", ctypes.c_int32), ("y", ctypes.c_void_p)]


class TensorDesc(ctypes.Structure):
    """nf4_tensor"""
    _fields_ = [("packed", ctypes.c_void_p), ("absmax", ctypes.c_void_p), ("dq", DQState),
                ("n", ctypes.c_int64), ("blocksize", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("out", ctypes.c_void_p)]


_lock = threading.Lock()
_lib = None


class NF4Error(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what} failed: {status_string(status)} ({status})")


def load() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = lib_path()
        if not os.path.exists(path):
            raise ImportError(f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(nvcc, sm_100a).  There is no CPU fallback.")
        lib = ctypes.CDLL(path)
        P, i64, i32, f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float
        st = ctypes.c_int
        sig = {
            "nf4_dequantize": ([P, P, ctypes.POINTER(DQState), i64, i32, i32, P, P], st),
            "nf4_dequantize_batched": ([ctypes.POINTER(TensorDesc), i32, i32, P], st),
            "nf4_dequantize_host": ([P, P, ctypes.POINTER(DQState), i64, i32, i32, P, P, i64, i64, P], st),
            "nf4_host_workspace_bytes": ([i64, i32, i32], i64),
            "nf4_dequantize_host_batched": ([ctypes.POINTER(TensorDesc), i32, i32, P, i64, i64, P], st),
            "nf4_quantize": ([P, i32, i64, i32, P, P, P], st),
            "nf4_double_quantize": ([P, i64, f32, P, i32, P, P, P], st),
            "nf4_codebook": ([P], None),
            "nf4_codebook_fp4": ([P], None),
            "nf4_gemm": ([P, i32, i32, P, P, ctypes.POINTER(DQState), i32, i32, i32, P, i32, i32, P, i64, P], st),
            "nf4_gemm_default_splits": ([i32, i32, i32], i32),
            "nf4_gemm_workspace_bytes": ([i32, i32, i32, i32], i64),
            "nf4_gemm_grouped": ([P, i32, i32, i32, i32, ctypes.POINTER(GemmWeight), i32, i32, P, i64, P], st),
            "nf4_gemm_grouped_workspace_bytes": ([i32, ctypes.POINTER(ctypes.c_int32), i32, i32], i64),
            "nf4_gemm_multi": ([ctypes.POINTER(GemmProblem), i32, i32, i32, i32, i32, P, i64, P], st),
            "nf4_gemm_multi_workspace_bytes": ([i32, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                                i32], i64),
            "nf4_gemm_set_early_weight_reads": ([i32], None),
            "nf4_set_early_input_reads": ([i32], None),
            "nf4_dequantize_ex": ([P, P, ctypes.POINTER(DQState), i64, i32, P, i32, P, P], st),
            "nf4_dequantize_batched_ex": ([ctypes.POINTER(TensorDesc), i32, P, i32, P], st),
            "nf4_status_string": ([st], ctypes.c_char_p),
            "nf4_last_launch_count": ([], i32),
            "nf4_synth_fill": ([i32, ctypes.c_uint64, i64, i64, P, P], st),
            "nf4_sol_stream": ([P, i64, P, P], st),
            "nf4_set_max_ctas": ([i32], None),
            "nf4_dequant_grid": ([i64], i32),
            "nf4_dequant_tile_elems": ([], i64),
            "nf4_kernel_variant_count": ([], i32),
            "nf4_kernel_variant_name": ([i32], ctypes.c_char_p),
            "nf4_set_kernel_variant": ([i32], i32),
            "nf4_get_kernel_variant": ([], i32),
        }
        for name, (args, res) in sig.items():
            if path != LIB_PATH and not hasattr(lib, name):
                continue          # diagnostics build of an older revision (NF4_LIB): skip newer symbols
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def status_string(s: int) -> str:
    return load().nf4_status_string(int(s)).decode()


def check(status: int, what: str) -> None:
    if status != NF4_OK:
        raise NF4Error(status, what)
