import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if not os.environ.get("NF4_LIB"):   # event traces / experiments need the diagnostics build
    from paper_2604_02556_b200 import _build
    os.environ["NF4_LIB"] = _build.build_variant("trace", {"NF4_GEMM_DIAG": 1})
import torch
import paper_2604_02556_b200 as nf4
from synth import stores
from synth import workloads as wl
M, N, K, S = 16, 21504, 5376, int(sys.argv[1]) if len(sys.argv) > 1 else 4
if len(sys.argv) > 4: M, N, K = map(int, sys.argv[2:5])
ws = stores.from_hash([wl.Tensor("w", N, K)], 64, True, "bf16", 3, "cuda")
e = ws.entries[0]
dq = nf4.DQ(ws._ptr(ws.scales, e.scale_off), ws.code2.data_ptr(), ws._ptr(ws.groups, e.group_off), e.offset)
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
wsp = torch.zeros(16 + nf4.nf4_gemm_workspace_bytes(M, N, K, S), dtype=torch.uint8, device="cuda")
tr = torch.zeros(1024 + 4 * 8192, dtype=torch.int64, device="cuda")
f = lambda: nf4.nf4_gemm(x, ws._ptr(ws.codes, e.codes_off), None, dq, N=N, K=K, y=y, splits=S, workspace=wsp)
for _ in range(3): f()
os.environ["NF4_GEMM_TRACE"] = str(tr.data_ptr())
torch.cuda.synchronize()
f(); torch.cuda.synchronize()
t = tr.cpu().numpy().astype('int64')
t0 = t[0]
print("CTA0 lifetime us", (t[1] - t0) / 1e3)
for j in range(8):
    if t[16 + j]: print(f"super {j}: tma_issue {(t[16+j]-t0)/1e3:7.2f}")

import numpy as np
c = t[1024:].reshape(-1, 4)
c = c[c[:, 0] > 0]
st, en, sm = (c[:, 0] - c[:, 0].min()) / 1e3, (c[:, 1] - c[:, 0].min()) / 1e3, c[:, 2]
print("CTAs", len(c), "kernel span us", en.max(), "start spread", np.percentile(st, [0, 25, 50, 75, 100]).round(2))
print("durations us p0/25/50/75/100", np.percentile(en - st, [0, 25, 50, 75, 100]).round(2))
ep = (c[:, 3] - c[:, 0].min()) / 1e3
print("end - last epilogue us p0/50/100", np.percentile(en - ep, [0, 50, 100]).round(2))
print("end times p0/25/50/75/100", np.percentile(en, [0, 25, 50, 75, 100]).round(2))
print("CTAs per SM (max concurrent)", np.bincount(sm.astype(int)).max(), "distinct SMs", len(set(sm.tolist())))
order = np.argsort(st)
print("first-wave starts (first 8):", st[order[:8]].round(2), "last 8 starts:", st[order[-8:]].round(2))
dur = en - st
cta = np.arange(len(c))
print("duration by CTA index decile:", [round(float(dur[(cta * 10 // len(c)) == d].mean()), 1) for d in range(10)])
sm_ids = sm.astype(int)
per_sm = np.array([dur[sm_ids == k].mean() if (sm_ids == k).any() else 0 for k in range(sm_ids.max() + 1)])
print("mean duration by SM id (groups of 16):", [round(float(per_sm[i:i + 16].mean()), 1) for i in range(0, len(per_sm), 16)])
print("per-SM mean p0/50/100:", np.percentile(per_sm[per_sm > 0], [0, 50, 100]).round(1))
# within-SM spread
spread = [dur[sm_ids == k].max() - dur[sm_ids == k].min() for k in set(sm_ids.tolist())]
print("within-SM spread p50/max:", np.percentile(spread, [50, 100]).round(1))
# slowest CTAs and their stream-K ranges (tile-major chunk stream, G = #CTAs)
if S == 0:
    nk = K // 64
    bn = 16 if M <= 16 else 32 if M <= 32 else 64 if M <= 64 else 128 if M <= 128 else 256
    tiles = -(-N // 128) * -(-M // bn)
    W, G = tiles * nk, len(c)
    a4 = nk % 4 == 0
    def bnd(cc):
        b = cc * W // G
        if a4:
            b = (b + 2) // 4 * 4
        return min(b, W)
    for idx in np.argsort(-dur)[:6]:
        x0, x1 = bnd(idx), bnd(idx + 1)
        print(f"CTA {idx}: {dur[idx]:.1f} us, start {st[idx]:.2f}, range [{x0},{x1}) tiles {x0 // nk}..{(x1 - 1) // nk}"
              f" kc0 {x0 % nk} end-in-tile {x1 - (x1 - 1) // nk * nk}")
