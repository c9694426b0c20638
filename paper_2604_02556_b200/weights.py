"""NF4 weight store: a model's quantized linear weights laid out flat in HBM.

Layout: one allocation per array kind --
packed codes (uint8), per-block scales (fp32 absmax, or uint8 qabsmax + fp32
absmax2), 16-bit outputs -- with each tensor's region starting on a 256-byte
boundary, so every tensor takes the library's vector path and a whole model is
dequantized by ceil(#tensors / NF4_MAX_BATCH) persistent launches of
nf4_dequantize_batched.  One fp32[256] second-level code table
is shared by all tensors; each tensor keeps its own DQ offset.

The synthetic builders that fill a store for the bench and the tests
(``from_hash``, ``from_gaussian``) live in ``synth/stores.py``: the product
package never imports the input generators.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

from . import DQ, NF4Tensor, nf4_dequantize_batched

ALIGN = 256


def _up(v: int, a: int = ALIGN) -> int:
    return (v + a - 1) // a * a


@dataclass
class Entry:
    name: str
    n: int
    seed: int
    codes_off: int
    scale_off: int       # bytes into the scale buffer (fp32 absmax or uint8 qabsmax)
    group_off: int       # bytes into absmax2 (DQ)
    out_off: int         # bytes into the output buffer
    offset: float = 0.0  # DQ offset


@dataclass
class WeightStore:
    blocksize: int
    dq: bool
    out_dtype: str
    entries: List[Entry] = field(default_factory=list)
    codes: object = None
    scales: object = None
    groups: object = None
    code2: object = None
    out: object = None

    # ------------------------------------------------------------------ sizes
    @property
    def n_total(self) -> int:
        return sum(e.n for e in self.entries)

    def algorithmic_bytes(self) -> int:
        """Bytes the method must move per pass: codes ceil(n/2),
        scales (4 B per block, or 1 B per block + 4 B per 256 blocks), 2 B/elt out."""
        tot = 0
        for e in self.entries:
            nb = -(-e.n // self.blocksize)
            tot += (e.n + 1) // 2 + 2 * e.n
            tot += (nb + 4 * (-(-nb // 256))) if self.dq else 4 * nb
        if self.dq and self.entries:
            tot += 1024  # code2, read once per pass
        return tot

    # --------------------------------------------------------------- layout
    @classmethod
    def layout(cls, tensors, blocksize: int, dq: bool, out_dtype: str, seed0: int, device):
        import torch
        ws = cls(blocksize, dq, out_dtype)
        co = so = go = oo = 0
        for i, t in enumerate(tensors):
            n = t.n
            nb = -(-n // blocksize)
            ws.entries.append(Entry(t.name, n, seed0 + i, co, so, go, oo))
            co += _up((n + 1) // 2)
            so += _up(nb if dq else 4 * nb)
            go += _up(4 * (-(-nb // 256))) if dq else 0
            oo += _up(2 * n)
        ws.codes = torch.empty(max(co, 1), dtype=torch.uint8, device=device)
        ws.scales = torch.empty(max(so, 1), dtype=torch.uint8, device=device)
        ws.groups = torch.empty(max(go, 4), dtype=torch.uint8, device=device)
        ws.out = torch.empty(max(oo, 2), dtype=torch.uint8, device=device)
        return ws

    def _ptr(self, buf, off):
        return buf.data_ptr() + off

    def nf4_tensors(self) -> List[NF4Tensor]:
        out = []
        for e in self.entries:
            if self.dq:
                dq = DQ(self._ptr(self.scales, e.scale_off), self.code2.data_ptr(),
                        self._ptr(self.groups, e.group_off), e.offset, 256)
                out.append(NF4Tensor(self._ptr(self.codes, e.codes_off), e.n, self.blocksize,
                                     self._ptr(self.out, e.out_off), None, dq))
            else:
                out.append(NF4Tensor(self._ptr(self.codes, e.codes_off), e.n, self.blocksize,
                                     self._ptr(self.out, e.out_off), self._ptr(self.scales, e.scale_off), None))
        return out

    # ------------------------------------------------------------ the path
    def dequantize_all(self, stream=None, descs=None) -> int:
        """One pass of the hot path over every tensor; returns kernels launched."""
        import paper_2604_02556_b200 as nf4
        nf4_dequantize_batched(descs if descs is not None else self.nf4_tensors(), self.out_dtype, stream)
        return nf4.nf4_last_launch_count()

    def out_view(self, i: int):
        import torch
        e = self.entries[i]
        dt = torch.float16 if self.out_dtype == "f16" else torch.bfloat16
        return self.out[e.out_off:e.out_off + 2 * e.n].view(dt)

    def out_words(self, i: int, k0: int, k1: int):
        """uint16 view of tensor i's outputs [k0, k1) (still on device)."""
        import torch
        e = self.entries[i]
        return self.out[e.out_off + 2 * k0:e.out_off + 2 * k1].view(torch.int16)
