#!/usr/bin/env python
"""ncu target: the F1 one-launch decode step (nf4_gemm_multi over the 56 linear
weights of 8 Gemma-3-27B layers, DQ, bf16) at M tokens, launched 3 times.

    ncu --set full --clock-control none --import-source on -k regex:nf4_gemm_kernel -s 2 -c 1 \
        python tools/gemm_prof_multi.py 16
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_02556_b200 as nf4
from synth import stores
from synth import workloads as wl

M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
torch.cuda.set_device(0)
tensors = wl.model_tensors("gemma-3-27b", layers=8)
ws = stores.from_hash(tensors, 64, True, "bf16", seed0=77, device="cuda")
xs = {}
for t in tensors:
    if t.cols not in xs:
        xs[t.cols] = torch.randn(M, t.cols, device="cuda").to(torch.bfloat16)
ys = [torch.empty(M, t.rows, dtype=torch.bfloat16, device="cuda") for t in tensors]
probs = []
for t, e in zip(tensors, ws.entries):
    dq = nf4.DQ(ws._ptr(ws.scales, e.scale_off), ws.code2.data_ptr(), ws._ptr(ws.groups, e.group_off), e.offset)
    probs.append((xs[t.cols], t.cols, ws._ptr(ws.codes, e.codes_off), None, dq, t.rows))
wsp = torch.zeros(max(16, nf4.nf4_gemm_multi_workspace_bytes(M, [t.rows for t in tensors], [t.cols for t in tensors])),
                  dtype=torch.uint8, device="cuda")
for _ in range(3):
    nf4.nf4_gemm_multi(probs, M=M, ys=ys, workspace=wsp)
torch.cuda.synchronize()
print("ok", sum(t.n for t in tensors), "weights")
