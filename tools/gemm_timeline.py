#!/usr/bin/env python
"""F1 launch timeline at production speed (NF4_GEMM_DIAG=1 build: globaltimer stamps,
no run-time experiment branches): one nf4_gemm launched right after an identical
untraced one (so it starts under programmatic dependent launch, as in a decode
loop), per-CTA start / end / last-epilogue times and CTA 0's first-stage events.

    python tools/gemm_timeline.py M N K
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if not os.environ.get("NF4_LIB"):
    from paper_2604_02556_b200 import _build
    os.environ["NF4_LIB"] = _build.build_variant("trace", {"NF4_GEMM_DIAG": 1})
import numpy as np
import torch

import paper_2604_02556_b200 as nf4
from synth import stores
from synth import workloads as wl

M, N, K = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (1, 43008, 5376)
torch.cuda.set_device(0)
ws = stores.from_hash([wl.Tensor("w", N, K)], 64, True, "bf16", 3, "cuda")
e = ws.entries[0]
dq = nf4.DQ(ws._ptr(ws.scales, e.scale_off), ws.code2.data_ptr(), ws._ptr(ws.groups, e.group_off), e.offset)
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
wsp = torch.zeros(16 + nf4.nf4_gemm_workspace_bytes(M, N, K, 0), dtype=torch.uint8, device="cuda")
tr = torch.zeros(1024 + 4 * 4096, dtype=torch.int64, device="cuda")
f = lambda: nf4.nf4_gemm(x, ws._ptr(ws.codes, e.codes_off), None, dq, N=N, K=K, y=y, splits=0, workspace=wsp)
out = {"M": M, "N": N, "K": K}
runs = []
for rep in range(5):
    for _ in range(3):
        f()
    os.environ.pop("NF4_GEMM_TRACE", None)
    f()                                          # untraced predecessor (PDL)
    os.environ["NF4_GEMM_TRACE"] = str(tr.data_ptr())
    f()                                          # traced launch
    os.environ.pop("NF4_GEMM_TRACE", None)
    torch.cuda.synchronize()
    t = tr.cpu().numpy().astype("int64")
    c = t[1024:].reshape(-1, 4)
    c = c[c[:, 0] > 0]
    t0 = c[:, 0].min()
    st, en, ep = (c[:, 0] - t0) / 1e3, (c[:, 1] - t0) / 1e3, (c[:, 3] - t0) / 1e3
    r = {"ctas": int(len(c)), "span_us": round(float(en.max()), 2),
         "start_spread_us": round(float(st.max()), 2),
         "duration_p0_50_100": np.percentile(en - st, [0, 50, 100]).round(2).tolist(),
         "end_p0_50_100": np.percentile(en, [0, 50, 100]).round(2).tolist(),
         "end_minus_last_epilogue_p50_max": np.percentile(en - ep, [50, 100]).round(2).tolist(),
         "cta0_after_wait_us": round(float((t[0] - t0) / 1e3), 2)}
    for name, base in (("prologue_table_built", 600), ("prologue_mbar_init", 603), ("prologue_init_fence", 604),
                       ("prologue_barriers_range", 601), ("prologue_tmem_alloc", 602),
                       ("first_codes_landed", 100), ("first_slot_free", 200), ("first_stage_done", 300),
                       ("first_x_issue", 400), ("first_mma", 500)):
        if t[base]:
            r[name + "_us"] = round(float((t[base] - t0) / 1e3), 2)
    runs.append(r)
    tr.zero_()
out["runs"] = runs
print(json.dumps(out))
