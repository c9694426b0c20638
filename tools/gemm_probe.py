#!/usr/bin/env python
"""Time one nf4_gemm shape across split-K factors (diagnostics for F1)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_02556_b200 as nf4
from synth import stores
from synth import workloads as wl

M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
N, K = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (4096, 5376)
torch.cuda.set_device(0)
ws = stores.from_hash([wl.Tensor("w", N, K)], 64, True, "bf16", 3, "cuda")
e = ws.entries[0]
dq = nf4.DQ(ws._ptr(ws.scales, e.scale_off), ws.code2.data_ptr(), ws._ptr(ws.groups, e.group_off), e.offset)
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
res = {}
for s in (0, 1, 2, 4, 8, 16, 32):
    wsp = torch.zeros(max(16, nf4.nf4_gemm_workspace_bytes(M, N, K, s)), dtype=torch.uint8, device="cuda")
    f = lambda: nf4.nf4_gemm(x, ws._ptr(ws.codes, e.codes_off), None, dq, N=N, K=K, y=y, splits=s, workspace=wsp)
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): f()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    res[s] = round(ms * 1000, 1)
print(json.dumps({"M": M, "N": N, "K": K, "us_by_splits": res, "ctas_split1": (N + 127) // 128}))
