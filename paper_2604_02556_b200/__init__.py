"""paper_2604_02556_b200 -- B200-native blockwise NF4 dequantization (arxiv 2604.02556).

Thin Python binding over libnf4.so (C-ABI: include/nf4.h, include/nf4_tools.h).
Functions carry the C names and only marshal arguments: torch is used for device
memory and streams; every step of the path runs in the library's sm_100a
kernels.  There is no CPU fallback: without the built library every call raises.

    import torch, paper_2604_02556_b200 as nf4
    packed, absmax = nf4.nf4_quantize(w, blocksize=64)            # inputs
    out = nf4.nf4_dequantize(packed, absmax, n=w.numel(), blocksize=64,
                             out_dtype=torch.float16)              # the hot path
"""
from __future__ import annotations

import ctypes
import functools
from dataclasses import dataclass
from typing import Optional, Sequence

from . import _lib
from ._lib import NF4Error, load, status_string  # noqa: F401

__all__ = [
    "DQ", "NF4Tensor", "NF4Error", "load", "status_string",
    "nf4_dequantize", "nf4_dequantize_batched", "nf4_dequantize_host", "nf4_host_workspace_bytes",
    "nf4_quantize", "nf4_double_quantize", "nf4_codebook", "nf4_last_launch_count",
    "nf4_synth_fill", "nf4_sol_stream", "nf4_set_max_ctas", "nf4_dequant_grid", "nf4_dequant_tile_elems",
    "nf4_kernel_variants", "nf4_set_kernel_variant", "nf4_get_kernel_variant",
    "nf4_dequantize_ex", "nf4_dequantize_batched_ex", "nf4_codebook_fp4",
    "nf4_gemm", "nf4_gemm_default_splits", "nf4_gemm_workspace_bytes", "nf4_dequantize_host_batched",
    "nf4_gemm_grouped", "nf4_gemm_grouped_workspace_bytes",
    "nf4_gemm_multi", "nf4_gemm_multi_workspace_bytes", "nf4_gemm_set_early_weight_reads",
    "nf4_set_early_input_reads",
]


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if hasattr(t, "data_ptr"):
        return t.data_ptr() if t.numel() > 0 else None
    if hasattr(t, "ctypes"):  # numpy
        return t.ctypes.data if t.size > 0 else None
    raise TypeError(f"cannot take a pointer of {type(t)}")


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)   # cheap (no Stream object)
        if raw is not None:
            return raw(torch.cuda.current_device()) or None
        return torch.cuda.current_stream().cuda_stream or None
    if isinstance(stream, int):
        return stream or None
    return stream.cuda_stream or None


def _dtype_code(dt) -> int:
    import torch
    if dt in (torch.float16, "f16", "fp16", _lib.NF4_F16):
        return _lib.NF4_F16
    if dt in (torch.bfloat16, "bf16", _lib.NF4_BF16):
        return _lib.NF4_BF16
    if dt in (torch.float32, "f32", "fp32", _lib.NF4_F32):
        return _lib.NF4_F32
    raise ValueError(f"unsupported dtype {dt}")


@dataclass
class DQ:
    """Double-quantized absmax state (nf4_dq_state): qabsmax uint8[nb], code2
    fp32[256], absmax2 fp32[ceil(nb/256)], offset, blocksize2 (= 256)."""
    qabsmax: object
    code2: object
    absmax2: object
    offset: float
    blocksize2: int = 256

    def c(self) -> _lib.DQState:
        return _lib.DQState(_ptr(self.qabsmax), _ptr(self.code2), _ptr(self.absmax2),
                            float(self.offset), int(self.blocksize2))


@dataclass
class NF4Tensor:
    """One tensor of a batched call (nf4_tensor)."""
    packed: object
    n: int
    blocksize: int
    out: object
    absmax: object = None
    dq: Optional[DQ] = None

    def c(self) -> _lib.TensorDesc:
        d = _lib.TensorDesc()
        d.packed = _ptr(self.packed)
        d.absmax = _ptr(self.absmax)
        d.dq = self.dq.c() if self.dq is not None else _lib.DQState(None, None, None, 0.0, 256)
        d.n = int(self.n)
        d.blocksize = int(self.blocksize)
        d.reserved = 0
        d.out = _ptr(self.out)
        return d


def nf4_dequantize(packed, absmax=None, dq: Optional[DQ] = None, *, n: int, blocksize: int = 64,
                   out_dtype="f16", out=None, stream=None):
    """out[k] = RNE16(fl32(NF4[code_k] * absmax_b)) for k < n (include/nf4.h).
    Allocates `out` with torch if not given; returns it."""
    import torch
    code = _dtype_code(out_dtype)
    if out is None:
        out = torch.empty(n, dtype=torch.float16 if code == _lib.NF4_F16 else torch.bfloat16,
                          device=packed.device)
    dqc = dq.c() if dq is not None else None
    st = load().nf4_dequantize(_ptr(packed), _ptr(absmax), ctypes.byref(dqc) if dqc is not None else None,
                               int(n), int(blocksize), code, _ptr(out), _stream(stream))
    _lib.check(st, "nf4_dequantize")
    return out


def _codebook_arg(codebook):
    if codebook is None:
        return None
    if isinstance(codebook, str):
        codebook = nf4_codebook_fp4() if codebook == "fp4" else nf4_codebook() if codebook == "nf4" else None
        if codebook is None:
            raise ValueError("codebook must be 'nf4', 'fp4' or 16 floats")
    vals = [float(v) for v in (codebook.tolist() if hasattr(codebook, "tolist") else codebook)]
    if len(vals) != 16:
        raise ValueError("codebook must have 16 entries")
    return (ctypes.c_float * 16)(*vals)


def nf4_dequantize_ex(packed, absmax=None, dq: Optional[DQ] = None, *, n: int, blocksize: int = 64,
                      codebook=None, out_dtype="f16", out=None, stream=None):
    """nf4_dequantize with another 16-entry codebook ('fp4', 'nf4' or 16 floats)
    and/or fp32 output."""
    import torch
    code = _dtype_code(out_dtype)
    if out is None:
        tdt = {_lib.NF4_F16: torch.float16, _lib.NF4_BF16: torch.bfloat16, _lib.NF4_F32: torch.float32}[code]
        out = torch.empty(n, dtype=tdt, device=packed.device)
    dqc = dq.c() if dq is not None else None
    st = load().nf4_dequantize_ex(_ptr(packed), _ptr(absmax), ctypes.byref(dqc) if dqc is not None else None,
                                  int(n), int(blocksize), _codebook_arg(codebook), code, _ptr(out), _stream(stream))
    _lib.check(st, "nf4_dequantize_ex")
    return out


def nf4_dequantize_batched_ex(tensors: Sequence[NF4Tensor], codebook=None, out_dtype="f16", stream=None) -> None:
    arr = (_lib.TensorDesc * max(len(tensors), 1))(*[t.c() for t in tensors])
    st = load().nf4_dequantize_batched_ex(arr, len(tensors), _codebook_arg(codebook), _dtype_code(out_dtype),
                                          _stream(stream))
    _lib.check(st, "nf4_dequantize_batched_ex")


def nf4_codebook_fp4():
    buf = (ctypes.c_float * 16)()
    load().nf4_codebook_fp4(buf)
    return list(buf)


def nf4_dequantize_batched(tensors: Sequence[NF4Tensor], out_dtype="f16", stream=None) -> None:
    arr = (_lib.TensorDesc * max(len(tensors), 1))(*[t.c() for t in tensors])
    st = load().nf4_dequantize_batched(arr, len(tensors), _dtype_code(out_dtype), _stream(stream))
    _lib.check(st, "nf4_dequantize_batched")


def nf4_host_workspace_bytes(chunk_elems: int, blocksize: int, dq: bool) -> int:
    return int(load().nf4_host_workspace_bytes(int(chunk_elems), int(blocksize), int(bool(dq))))


def nf4_dequantize_host(packed, absmax=None, dq: Optional[DQ] = None, *, n: int, blocksize: int = 64,
                        out_dtype="f16", out, workspace, chunk_elems: int, stream=None) -> None:
    """Host-buffer end-to-end path: all array arguments are host (ideally pinned)
    tensors/arrays; `workspace` is a device buffer of nf4_host_workspace_bytes()."""
    dqc = dq.c() if dq is not None else None
    nbytes = workspace.numel() * workspace.element_size()
    st = load().nf4_dequantize_host(_ptr(packed), _ptr(absmax), ctypes.byref(dqc) if dqc is not None else None,
                                    int(n), int(blocksize), _dtype_code(out_dtype), _ptr(out), _ptr(workspace),
                                    int(nbytes), int(chunk_elems), _stream(stream))
    _lib.check(st, "nf4_dequantize_host")


def nf4_dequantize_host_batched(tensors: Sequence[NF4Tensor], out_dtype="f16", *, workspace, chunk_elems: int,
                                stream=None) -> None:
    """Host-buffer path over several tensors in one pipeline (all descriptor
    pointers are host memory; `workspace` is a device buffer)."""
    arr = (_lib.TensorDesc * max(len(tensors), 1))(*[t.c() for t in tensors])
    nbytes = workspace.numel() * workspace.element_size()
    st = load().nf4_dequantize_host_batched(arr, len(tensors), _dtype_code(out_dtype), _ptr(workspace), int(nbytes),
                                            int(chunk_elems), _stream(stream))
    _lib.check(st, "nf4_dequantize_host_batched")


def nf4_quantize(x, blocksize: int = 64, packed=None, absmax=None, stream=None):
    """GPU NF4 quantizer (input generator).  x: CUDA tensor f32/f16/bf16.
    Returns (packed uint8[ceil(n/2)], absmax fp32[ceil(n/blocksize)])."""
    import torch
    n = x.numel()
    if packed is None:
        packed = torch.empty((n + 1) // 2, dtype=torch.uint8, device=x.device)
    if absmax is None:
        absmax = torch.empty(-(-n // blocksize), dtype=torch.float32, device=x.device)
    st = load().nf4_quantize(_ptr(x), _dtype_code(x.dtype), n, int(blocksize), _ptr(packed), _ptr(absmax),
                             _stream(stream))
    _lib.check(st, "nf4_quantize")
    return packed, absmax


def nf4_double_quantize(absmax, offset: float, code2, qabsmax=None, absmax2=None, blocksize2: int = 256,
                        stream=None) -> DQ:
    """GPU second-level quantizer (input generator).  Returns the DQ state."""
    import torch
    nb = absmax.numel()
    if qabsmax is None:
        qabsmax = torch.empty(nb, dtype=torch.uint8, device=absmax.device)
    if absmax2 is None:
        absmax2 = torch.empty(-(-nb // blocksize2), dtype=torch.float32, device=absmax.device)
    st = load().nf4_double_quantize(_ptr(absmax), nb, float(offset), _ptr(code2), int(blocksize2), _ptr(qabsmax),
                                    _ptr(absmax2), _stream(stream))
    _lib.check(st, "nf4_double_quantize")
    return DQ(qabsmax, code2, absmax2, float(offset), blocksize2)


def nf4_codebook():
    buf = (ctypes.c_float * 16)()
    load().nf4_codebook(buf)
    return list(buf)


def nf4_last_launch_count() -> int:
    return int(load().nf4_last_launch_count())


def nf4_synth_fill(kind: int, seed: int, begin: int, count: int, dst, stream=None) -> None:
    st = load().nf4_synth_fill(int(kind), int(seed), int(begin), int(count), _ptr(dst), _stream(stream))
    _lib.check(st, "nf4_synth_fill")


def nf4_sol_stream(src, in_bytes: int, dst, stream=None) -> None:
    st = load().nf4_sol_stream(_ptr(src), int(in_bytes), _ptr(dst), _stream(stream))
    _lib.check(st, "nf4_sol_stream")


def nf4_set_max_ctas(max_ctas: int) -> None:
    load().nf4_set_max_ctas(int(max_ctas))


def nf4_dequant_grid(tiles: int) -> int:
    return int(load().nf4_dequant_grid(int(tiles)))


def nf4_dequant_tile_elems() -> int:
    return int(load().nf4_dequant_tile_elems())


def nf4_kernel_variants():
    lib = load()
    return [lib.nf4_kernel_variant_name(i).decode() for i in range(lib.nf4_kernel_variant_count())]


def nf4_set_kernel_variant(v) -> int:
    """Select the dequant kernel variant by index or name; returns the one in effect."""
    if isinstance(v, str):
        v = nf4_kernel_variants().index(v)
    return int(load().nf4_set_kernel_variant(int(v)))


def nf4_get_kernel_variant() -> int:
    return int(load().nf4_get_kernel_variant())


# ---------------------------------------------------------------------------
# F1: fused NF4 dequant + tcgen05 GEMM (include/nf4_gemm.h)
# ---------------------------------------------------------------------------
def nf4_gemm_default_splits(M: int, N: int, K: int) -> int:
    return int(load().nf4_gemm_default_splits(int(M), int(N), int(K)))


@functools.lru_cache(maxsize=4096)
def nf4_gemm_workspace_bytes(M: int, N: int, K: int, splits: int) -> int:
    return int(load().nf4_gemm_workspace_bytes(int(M), int(N), int(K), int(splits)))


def nf4_gemm(x, packed, absmax=None, dq: Optional[DQ] = None, *, N: int, K: int, blocksize: int = 64,
             y=None, y_dtype="bf16", splits: int = 0, workspace=None, stream=None):
    """Y = X . W^T with W the NF4 weight [N, K] dequantized on the fly.
    x: CUDA tensor [M, K] bf16/fp16.  splits <= 0: stream-K over all resident CTAs
    (default); splits >= 1: classic split-K grid.  Allocates y (and the partial-sum
    workspace) with torch when not given; returns y."""
    import torch
    M = x.shape[0] if x.dim() == 2 else x.numel() // K
    ycode = _dtype_code(y_dtype)
    if y is None:
        tdt = {_lib.NF4_F16: torch.float16, _lib.NF4_BF16: torch.bfloat16, _lib.NF4_F32: torch.float32}[ycode]
        y = torch.empty((M, N), dtype=tdt, device=x.device)
    if splits < 0:
        splits = 0
    wbytes = nf4_gemm_workspace_bytes(M, N, K, splits)
    if wbytes > 0 and workspace is None:
        workspace = torch.zeros(wbytes, dtype=torch.uint8, device=x.device)   # stream-K counters start at 0
    wsize = 0 if workspace is None else workspace.numel() * workspace.element_size()
    dqc = dq.c() if dq is not None else None
    st = load().nf4_gemm(_ptr(x), _dtype_code(x.dtype), int(M), _ptr(packed), _ptr(absmax),
                         ctypes.byref(dqc) if dqc is not None else None, int(N), int(K), int(blocksize),
                         _ptr(y), ycode, int(splits), _ptr(workspace), int(wsize), _stream(stream))
    _lib.check(st, "nf4_gemm")
    return y


@functools.lru_cache(maxsize=4096)
def nf4_gemm_grouped_workspace_bytes(M: int, Ns: tuple, K: int) -> int:
    arr = (ctypes.c_int32 * len(Ns))(*[int(n) for n in Ns])
    return int(load().nf4_gemm_grouped_workspace_bytes(int(M), arr, len(Ns), int(K)))


def nf4_gemm_grouped(x, weights, *, K: int, blocksize: int = 64, ys=None, y_dtype="bf16", workspace=None,
                     stream=None):
    """Y_i = X . W_i^T for up to 4 NF4 weights sharing X (e.g. q/k/v) in one stream-K
    launch (include/nf4_gemm.h).  weights: sequence of (packed, absmax, dq, N);
    returns the list of y_i [M, N_i] (allocated with torch unless `ys` is given)."""
    import torch
    M = x.shape[0] if x.dim() == 2 else x.numel() // K
    ycode = _dtype_code(y_dtype)
    tdt = {_lib.NF4_F16: torch.float16, _lib.NF4_BF16: torch.bfloat16, _lib.NF4_F32: torch.float32}[ycode]
    if ys is None:
        ys = [torch.empty((M, int(w[3])), dtype=tdt, device=x.device) for w in weights]
    Ns = tuple(int(w[3]) for w in weights)
    wbytes = nf4_gemm_grouped_workspace_bytes(M, Ns, K)
    if wbytes > 0 and workspace is None:
        workspace = torch.zeros(wbytes, dtype=torch.uint8, device=x.device)
    wsize = 0 if workspace is None else workspace.numel() * workspace.element_size()
    arr = (_lib.GemmWeight * len(weights))()
    for i, (packed, absmax, dq, n) in enumerate(weights):
        arr[i].packed = _ptr(packed)
        arr[i].absmax = _ptr(absmax)
        if dq is not None:
            arr[i].dq = dq.c()
        arr[i].N = int(n)
        arr[i].y = _ptr(ys[i])
    st = load().nf4_gemm_grouped(_ptr(x), _dtype_code(x.dtype), int(M), int(K), int(blocksize), arr, len(weights),
                                 ycode, _ptr(workspace), int(wsize), _stream(stream))
    _lib.check(st, "nf4_gemm_grouped")
    return ys


def nf4_gemm_multi_workspace_bytes(M: int, Ns, Ks) -> int:
    Ns, Ks = tuple(int(n) for n in Ns), tuple(int(k) for k in Ks)
    return _multi_ws_bytes(int(M), Ns, Ks)


@functools.lru_cache(maxsize=4096)
def _multi_ws_bytes(M: int, Ns: tuple, Ks: tuple) -> int:
    na = (ctypes.c_int32 * len(Ns))(*Ns)
    ka = (ctypes.c_int32 * len(Ks))(*Ks)
    return int(load().nf4_gemm_multi_workspace_bytes(M, na, ka, len(Ns)))


def nf4_gemm_multi(problems, *, M: int, blocksize: int = 64, x_dtype="bf16", y_dtype="bf16", ys=None,
                   workspace=None, stream=None):
    """Y_i = X_i . W_i^T for up to NF4_GEMM_MAX_MULTI independent problems in ONE
    persistent stream-K launch (include/nf4_gemm.h).  problems: sequence of
    (x [M, K_i], K_i, packed, absmax, dq, N_i).  Returns the list of y_i [M, N_i]
    (allocated with torch unless `ys` is given)."""
    import torch
    ycode = _dtype_code(y_dtype)
    tdt = {_lib.NF4_F16: torch.float16, _lib.NF4_BF16: torch.bfloat16, _lib.NF4_F32: torch.float32}[ycode]
    if ys is None:
        dev = next((q[0].device for q in problems if hasattr(q[0], "device")), None)
        ys = [torch.empty((M, int(q[5])), dtype=tdt, device=dev) for q in problems]
    Ns = tuple(int(q[5]) for q in problems)
    Ks = tuple(int(q[1]) for q in problems)
    wbytes = _multi_ws_bytes(int(M), Ns, Ks)
    if wbytes > 0 and workspace is None:
        workspace = torch.zeros(wbytes, dtype=torch.uint8, device=ys[0].device)
    wsize = 0 if workspace is None else workspace.numel() * workspace.element_size()
    arr = (_lib.GemmProblem * len(problems))()
    for i, (x, K, packed, absmax, dq, n) in enumerate(problems):
        arr[i].x = _ptr(x)
        arr[i].K = int(K)
        arr[i].packed = _ptr(packed)
        arr[i].absmax = _ptr(absmax)
        if dq is not None:
            arr[i].dq = dq.c()
        arr[i].N = int(n)
        arr[i].y = _ptr(ys[i])
    st = load().nf4_gemm_multi(arr, len(problems), int(M), _dtype_code(x_dtype), int(blocksize), ycode,
                               _ptr(workspace), int(wsize), _stream(stream))
    _lib.check(st, "nf4_gemm_multi")
    return ys


def nf4_gemm_set_early_weight_reads(enable: bool) -> None:
    load().nf4_gemm_set_early_weight_reads(1 if enable else 0)


def nf4_set_early_input_reads(enable: bool) -> None:
    """Dequantization kernels read their inputs before waiting for the previous
    kernel on the stream (contract in include/nf4.h); default off."""
    load().nf4_set_early_input_reads(1 if enable else 0)
