"""NF4Linear: a drop-in quantized linear layer on top of the C-ABI (the paper's
"standard quantized linear layer API", re-built B200-native).

The weight [out_features, in_features] is stored as BNB-format NF4 codes with
blockwise absmax (double-quantized by default, QLoRA's format).  forward():

* decode-size inputs (M = tokens <= ``fused_max_m``) run the fused NF4 dequant +
  tcgen05 GEMM (``nf4_gemm``): the 16-bit weight never exists in HBM;
* larger M (prefill) dequantize once with ``nf4_dequantize`` into a reusable
  buffer and use a library GEMM (cuBLAS via torch.matmul).

Both paths use exactly the hot path's weight values (bit-exact to the oracle).
"""
from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import DQ, nf4_dequantize, nf4_double_quantize, nf4_gemm, nf4_gemm_workspace_bytes, nf4_quantize


class NF4Linear(torch.nn.Module):
    def __init__(self, in_features: int, out_features: int, blocksize: int = 64, double_quant: bool = True,
                 compute_dtype: torch.dtype = torch.bfloat16, device=None, fused_max_m: int = 128,
                 bias: bool = False):
        super().__init__()
        if compute_dtype not in (torch.bfloat16, torch.float16):
            raise ValueError("compute_dtype must be bfloat16 or float16")
        self.in_features, self.out_features = in_features, out_features
        self.blocksize, self.double_quant = blocksize, double_quant
        self.compute_dtype = compute_dtype
        self.fused_max_m = fused_max_m
        n = in_features * out_features
        nb = -(-n // blocksize)
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.register_buffer("packed", torch.zeros((n + 1) // 2, dtype=torch.uint8, device=dev))
        if double_quant:
            self.register_buffer("qabsmax", torch.zeros(nb, dtype=torch.uint8, device=dev))
            self.register_buffer("absmax2", torch.zeros(-(-nb // 256), dtype=torch.float32, device=dev))
            self.register_buffer("code2", torch.zeros(256, dtype=torch.float32, device=dev))
            # the DQ offset is state (saved / loaded with the weights); `offset` is its
            # host copy, so forward never syncs to read it
            self.register_buffer("dq_offset", torch.zeros((), dtype=torch.float32, device=dev))
            self.offset = 0.0
            self.absmax = None
        else:
            self.register_buffer("absmax", torch.zeros(nb, dtype=torch.float32, device=dev))
        self.register_buffer("bias", torch.zeros(out_features, dtype=compute_dtype, device=dev) if bias else None)
        self._wbuf: Optional[torch.Tensor] = None
        self._gemm_ws: dict = {}     # M -> zero-initialised stream-K workspace (kept zeroed by nf4_gemm)

    # ------------------------------------------------------------------ build
    @classmethod
    def from_weight(cls, weight: torch.Tensor, bias: Optional[torch.Tensor] = None, blocksize: int = 64,
                    double_quant: bool = True, compute_dtype: torch.dtype = torch.bfloat16,
                    code2: Optional[torch.Tensor] = None, fused_max_m: int = 128) -> "NF4Linear":
        """Quantize a dense [out, in] weight on the GPU (nf4_quantize, + nf4_double_quantize
        with offset = mean(absmax) and the BNB signed dynamic code table by default)."""
        out_f, in_f = weight.shape
        m = cls(in_f, out_f, blocksize, double_quant, compute_dtype, weight.device, fused_max_m, bias is not None)
        w = weight.detach().contiguous()
        if w.dtype not in (torch.float32, torch.float16, torch.bfloat16):
            w = w.float()
        if double_quant:
            absmax = torch.empty(m.qabsmax.numel(), dtype=torch.float32, device=w.device)
            nf4_quantize(w.reshape(-1), blocksize, packed=m.packed, absmax=absmax)
            if code2 is None:
                from .tables import bnb_dynamic_code2  # the BNB table is plain data (an input)
                code2 = torch.from_numpy(bnb_dynamic_code2())
            m.code2.copy_(code2.to(device=w.device, dtype=torch.float32))
            m.offset = float(np.float32(absmax.double().mean().item()))
            m.dq_offset.fill_(m.offset)
            nf4_double_quantize(absmax, m.offset, m.code2, qabsmax=m.qabsmax, absmax2=m.absmax2)
        else:
            nf4_quantize(w.reshape(-1), blocksize, packed=m.packed, absmax=m.absmax)
        if bias is not None:
            m.bias.copy_(bias.detach().to(compute_dtype))
        return m

    def _load_from_state_dict(self, state_dict, prefix, *args, **kwargs):
        super()._load_from_state_dict(state_dict, prefix, *args, **kwargs)
        if self.double_quant:
            self.offset = float(self.dq_offset)

    def _dq(self) -> Optional[DQ]:
        return DQ(self.qabsmax, self.code2, self.absmax2, self.offset) if self.double_quant else None

    # --------------------------------------------------------------- compute
    def dequantize(self, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """The dense weight [out, in] in compute_dtype (the hot path, bit-exact)."""
        n = self.in_features * self.out_features
        w = nf4_dequantize(self.packed, self.absmax, self._dq(), n=n, blocksize=self.blocksize,
                           out_dtype=self.compute_dtype, out=out)
        return w.view(self.out_features, self.in_features)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        shape = x.shape
        x2 = x.reshape(-1, self.in_features).to(self.compute_dtype).contiguous()
        M, K = x2.shape
        fused_ok = (K % 64 == 0 and K % self.blocksize == 0 and x2.data_ptr() % 16 == 0
                    and self.packed.data_ptr() % 16 == 0)
        if M <= self.fused_max_m and fused_ok:
            ws = self._gemm_ws.get(M)
            if ws is None:
                nbytes = nf4_gemm_workspace_bytes(M, self.out_features, K, 0)
                ws = self._gemm_ws[M] = torch.zeros(max(nbytes, 16), dtype=torch.uint8, device=x.device)
            y = nf4_gemm(x2, self.packed, self.absmax, self._dq(), N=self.out_features, K=K,
                         blocksize=self.blocksize, y_dtype=self.compute_dtype, workspace=ws)
        else:
            if self._wbuf is None or self._wbuf.numel() != self.in_features * self.out_features:
                self._wbuf = torch.empty(self.in_features * self.out_features, dtype=self.compute_dtype,
                                         device=x.device)
            y = x2 @ self.dequantize(self._wbuf).t()
        if self.bias is not None:
            y = y + self.bias
        return y.reshape(*shape[:-1], self.out_features)

    def extra_repr(self) -> str:
        return (f"in_features={self.in_features}, out_features={self.out_features}, blocksize={self.blocksize}, "
                f"double_quant={self.double_quant}, compute_dtype={self.compute_dtype}")


class NF4LinearGroup(torch.nn.Module):
    """Up to 4 NF4Linear layers that consume the same input (q/k/v, gate/up): one
    ``nf4_gemm_grouped`` launch for decode-size inputs, so the fused kernel's
    fill/drain is paid once per group.  Larger M falls back to the
    members' own forward.  Returns a list with one output per member."""

    def __init__(self, members, fused_max_m: int = 256):
        super().__init__()
        self.fused_max_m = fused_max_m   # grouped fused beats dequantize+cuBLAS up to M = 256 (r01)
        members = list(members)
        if not 1 <= len(members) <= 4:
            raise ValueError("1..4 members")
        k = members[0].in_features
        if any(m.in_features != k or m.blocksize != members[0].blocksize or
               m.compute_dtype != members[0].compute_dtype for m in members):
            raise ValueError("members must share in_features, blocksize and compute_dtype")
        self.members = torch.nn.ModuleList(members)
        self._ws: dict = {}

    def forward(self, x: torch.Tensor):
        from . import nf4_gemm_grouped, nf4_gemm_grouped_workspace_bytes
        m0 = self.members[0]
        shape = x.shape
        x2 = x.reshape(-1, m0.in_features).to(m0.compute_dtype).contiguous()
        M, K = x2.shape
        fused_ok = (M <= self.fused_max_m and K % 64 == 0 and K % m0.blocksize == 0 and x2.data_ptr() % 16 == 0
                    and all(m.packed.data_ptr() % 16 == 0 for m in self.members))
        if not fused_ok:
            return [m(x) for m in self.members]
        Ns = tuple(m.out_features for m in self.members)
        ws = self._ws.get(M)
        if ws is None:
            nbytes = nf4_gemm_grouped_workspace_bytes(M, Ns, K)
            ws = self._ws[M] = torch.zeros(max(nbytes, 16), dtype=torch.uint8, device=x.device)
        weights = [(m.packed, m.absmax, m._dq(), m.out_features) for m in self.members]
        ys = nf4_gemm_grouped(x2, weights, K=K, blocksize=m0.blocksize, y_dtype=m0.compute_dtype, workspace=ws)
        out = []
        for m, y in zip(self.members, ys):
            if m.bias is not None:
                y = y + m.bias
            out.append(y.reshape(*shape[:-1], m.out_features))
        return out
