import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2604_02556_b200 as nf4
from synth import stores
from synth import workloads as wl
M, N, K, S = 16, 21504, 5376, int(sys.argv[1]) if len(sys.argv) > 1 else 0
if len(sys.argv) > 4:
    M, N, K = (int(v) for v in sys.argv[2:5])
ws = stores.from_hash([wl.Tensor("w", N, K)], 64, True, "bf16", 3, "cuda")
e = ws.entries[0]
dq = nf4.DQ(ws._ptr(ws.scales, e.scale_off), ws.code2.data_ptr(), ws._ptr(ws.groups, e.group_off), e.offset)
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
wsp = torch.zeros(16 + nf4.nf4_gemm_workspace_bytes(M, N, K, S), dtype=torch.uint8, device="cuda")
for _ in range(3):
    nf4.nf4_gemm(x, ws._ptr(ws.codes, e.codes_off), None, dq, N=N, K=K, y=y, splits=S, workspace=wsp)
torch.cuda.synchronize()
