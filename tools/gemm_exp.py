#!/usr/bin/env python
"""F1 diagnostics: one nf4_gemm shape, stream-K, timed (a) as a plain launch loop
(host overhead included when the GPU starves) and (b) replayed from a CUDA graph
(GPU time only), for the NF4_GEMM_EXPERIMENT knobs: 0 full kernel, 1 skip MMA,
2 skip dequant, 4 skip tcgen05.st, and combinations.

    python tools/gemm_exp.py 16 21504 5376
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
_exps_arg = sys.argv[4] if len(sys.argv) > 4 else "0,1,2,4,6,7"
if not os.environ.get("NF4_LIB") and _exps_arg != "0":
    # pipeline-skipping experiments need the diagnostics build (itself ~2x slower: its
    # numbers compare experiments with each other, not with the production library)
    from paper_2604_02556_b200 import _build
    os.environ["NF4_LIB"] = _build.build_variant("exp", {"NF4_GEMM_DIAG": 2})
import torch

import paper_2604_02556_b200 as nf4
from synth import stores
from synth import workloads as wl

M, N, K = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (16, 21504, 5376)
exps = [int(v) for v in sys.argv[4].split(",")] if len(sys.argv) > 4 else [0, 1, 2, 4, 6, 7]
torch.cuda.set_device(0)
ws = stores.from_hash([wl.Tensor("w", N, K)], 64, True, "bf16", 3, "cuda")
e = ws.entries[0]
dq = nf4.DQ(ws._ptr(ws.scales, e.scale_off), ws.code2.data_ptr(), ws._ptr(ws.groups, e.group_off), e.offset)
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
wsp = torch.zeros(max(16, nf4.nf4_gemm_workspace_bytes(M, N, K, 0)), dtype=torch.uint8, device="cuda")
f = lambda: nf4.nf4_gemm(x, ws._ptr(ws.codes, e.codes_off), None, dq, N=N, K=K, y=y, splits=0, workspace=wsp)
res = {"M": M, "N": N, "K": K}
s = torch.cuda.Stream()
for ex in exps:
    os.environ["NF4_GEMM_EXPERIMENT"] = str(ex)
    with torch.cuda.stream(s):
        for _ in range(3):
            f()
        s.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        import time
        a.record(s)
        t0 = time.perf_counter()
        for _ in range(20):
            f()
        host_us = (time.perf_counter() - t0) / 20 * 1e6
        b.record(s)
        s.synchronize()
        loop_us = a.elapsed_time(b) / 20 * 1e3
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                f()
        g.replay()
        s.synchronize()
        a.record(s)
        g.replay()
        b.record(s)
        s.synchronize()
        graph_us = a.elapsed_time(b) / 20 * 1e3
    res[f"exp{ex}"] = {"loop_us": round(loop_us, 1), "graph_us": round(graph_us, 1), "host_us": round(host_us, 1)}
os.environ.pop("NF4_GEMM_EXPERIMENT")
# host cost of the bare C call (arguments marshalled once)
import ctypes
import time
lib = nf4.load()
dqc = dq.c()
args = (x.data_ptr(), 1, M, ws._ptr(ws.codes, e.codes_off), None, ctypes.byref(dqc), N, K, 64, y.data_ptr(), 1, 0,
        wsp.data_ptr(), wsp.numel(), None)
for _ in range(3):
    lib.nf4_gemm(*args)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    lib.nf4_gemm(*args)
res["c_call_host_us"] = round((time.perf_counter() - t0) / 20 * 1e6, 1)
torch.cuda.synchronize()
print(json.dumps(res))
