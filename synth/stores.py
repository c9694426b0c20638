"""Fill a WeightStore (paper_2604_02556_b200.weights) with synthetic inputs.

Input generation only (no dequantization arithmetic):
  * ``from_hash``     -- counter-based synthetic codes/scales (synth.inputs streams,
                         written on the device by the library's nf4_synth_fill), the
                         same values the host oracle can regenerate at any index;
  * ``from_gaussian`` -- W ~ N(0, 0.02^2) drawn on the device with torch, then
                         quantized by the library's nf4_quantize (+ nf4_double_quantize).
"""
from __future__ import annotations

import numpy as np

from paper_2604_02556_b200 import _lib, nf4_double_quantize, nf4_quantize, nf4_synth_fill
from paper_2604_02556_b200.weights import WeightStore


def from_hash(tensors, blocksize: int, dq: bool, out_dtype: str, seed0: int, device, code2=None) -> WeightStore:
    """Synthetic counter-based inputs (synth.inputs streams), generated on device."""
    import torch
    from synth import inputs as syn
    ws = WeightStore.layout(tensors, blocksize, dq, out_dtype, seed0, device)
    if dq:
        c2 = syn.dynamic_map_code2() if code2 is None else code2
        ws.code2 = torch.from_numpy(np.ascontiguousarray(c2, np.float32)).to(device)
    for e in ws.entries:
        nb = -(-e.n // blocksize)
        nf4_synth_fill(_lib.NF4_SYNTH_CODES, e.seed, 0, (e.n + 1) // 2, ws._ptr(ws.codes, e.codes_off))
        if dq:
            nf4_synth_fill(_lib.NF4_SYNTH_QABSMAX, e.seed, 0, nb, ws._ptr(ws.scales, e.scale_off))
            nf4_synth_fill(_lib.NF4_SYNTH_ABSMAX2, e.seed, 0, -(-nb // 256), ws._ptr(ws.groups, e.group_off))
            e.offset = float(syn.hash_offset(e.seed))
        else:
            nf4_synth_fill(_lib.NF4_SYNTH_ABSMAX, e.seed, 0, nb, ws._ptr(ws.scales, e.scale_off))
    return ws


def from_gaussian(tensors, blocksize: int, dq: bool, out_dtype: str, seed0: int, device,
                  std: float = 0.02, code2=None) -> WeightStore:
    """W ~ N(0, std^2) per tensor on the device, quantized by nf4_quantize; DQ
    offset = mean(absmax) (fp64 accumulate), then nf4_double_quantize."""
    import torch
    from synth import inputs as syn
    ws = WeightStore.layout(tensors, blocksize, dq, out_dtype, seed0, device)
    if dq:
        c2 = syn.dynamic_map_code2() if code2 is None else code2
        ws.code2 = torch.from_numpy(np.ascontiguousarray(c2, np.float32)).to(device)
    g = torch.Generator(device=device)
    for e in ws.entries:
        g.manual_seed(e.seed)
        w = torch.randn(e.n, generator=g, device=device, dtype=torch.float32).mul_(std)
        nb = -(-e.n // blocksize)
        packed = ws.codes[e.codes_off:e.codes_off + (e.n + 1) // 2]
        if dq:
            absmax = torch.empty(nb, dtype=torch.float32, device=device)
            nf4_quantize(w, blocksize, packed=packed, absmax=absmax)
            e.offset = float(np.float32(absmax.double().mean().item()))
            q = ws.scales[e.scale_off:e.scale_off + nb]
            a2 = ws.groups[e.group_off:e.group_off + 4 * (-(-nb // 256))].view(torch.float32)
            nf4_double_quantize(absmax, e.offset, ws.code2, qabsmax=q, absmax2=a2)
            del absmax
        else:
            absmax = ws.scales[e.scale_off:e.scale_off + 4 * nb].view(torch.float32)
            nf4_quantize(w, blocksize, packed=packed, absmax=absmax)
        del w
    return ws
