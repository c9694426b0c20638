#!/usr/bin/env python
"""F1 diagnostics: per-super-stage event times (us from kernel start) of CTA 0 of a
stream-K nf4_gemm launch: TMA issue, group c_full seen, group a_free seen, group
w_full arrive, MMA w_full seen.   python tools/gemm_trace2.py M N K [experiment]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
if not os.environ.get("NF4_LIB"):   # event traces / experiments need the diagnostics build
    from paper_2604_02556_b200 import _build
    os.environ["NF4_LIB"] = _build.build_variant("trace", {"NF4_GEMM_DIAG": 1})
import torch

import paper_2604_02556_b200 as nf4
from synth import stores
from synth import workloads as wl

M, N, K = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (16, 21504, 5376)
if len(sys.argv) > 4:
    os.environ["NF4_GEMM_EXPERIMENT"] = sys.argv[4]
ws = stores.from_hash([wl.Tensor("w", N, K)], 64, True, "bf16", 3, "cuda")
e = ws.entries[0]
dq = nf4.DQ(ws._ptr(ws.scales, e.scale_off), ws.code2.data_ptr(), ws._ptr(ws.groups, e.group_off), e.offset)
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
wsp = torch.zeros(16 + nf4.nf4_gemm_workspace_bytes(M, N, K, 0), dtype=torch.uint8, device="cuda")
tr = torch.zeros(1024 + 4 * 8192, dtype=torch.int64, device="cuda")
f = lambda: nf4.nf4_gemm(x, ws._ptr(ws.codes, e.codes_off), None, dq, N=N, K=K, y=y, splits=0, workspace=wsp)
for _ in range(3):
    f()
os.environ["NF4_GEMM_TRACE"] = str(tr.data_ptr())
torch.cuda.synchronize()
f()
torch.cuda.synchronize()
t = tr.cpu().numpy().astype(np.int64)
t0 = t[0]
c = t[1024:].reshape(-1, 4)
c = c[c[:, 0] > 0]
print("CTA0 lifetime us", (c[0, 1] - c[0, 0]) / 1e3, " kernel span", (c[:, 1].max() - c[:, 0].min()) / 1e3)
print(" J   tma   cfull  afree  wfull  mma")
for J in range(80):
    if t[400 + J] == 0:
        break
    row = [t[400 + J], t[100 + J], t[200 + J], t[300 + J], t[500 + J]]
    print(f"{J:2d} " + " ".join(f"{(v - t0) / 1e3:6.2f}" if v else "   -  " for v in row))
