#!/usr/bin/env python
"""One nf4_gemm / nf4_gemm_multi call on counter-hash weights (diagnostics):
    python tools/gemm_case.py M N K blocksize dq splits|multi"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2604_02556_b200 as nf4
from synth import inputs as syn

M, N, K, bs, dq = (int(v) for v in sys.argv[1:6])
mode = sys.argv[6]
n = N * K
nb = n // bs
packed = torch.from_numpy(syn.hash_packed(1, 0, n // 2)).cuda()
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
if dq:
    d = nf4.DQ(torch.from_numpy(syn.hash_qabsmax(1, 0, nb)).cuda(), torch.from_numpy(syn.dynamic_map_code2()).cuda(),
               torch.from_numpy(syn.hash_absmax2(1, 0, -(-nb // 256))).cuda(), 0.05)
    a = None
else:
    d, a = None, torch.from_numpy(syn.hash_absmax(1, 0, nb)).cuda()
if mode == "multi":
    ys = nf4.nf4_gemm_multi([(x, K, packed, a, d, N)] * 2, M=M, blocksize=bs, y_dtype="f32")
else:
    ys = [nf4.nf4_gemm(x, packed, a, d, N=N, K=K, blocksize=bs, y_dtype="f32", splits=int(mode))]
torch.cuda.synchronize()
print("ok", mode, float(ys[0].abs().sum()))
