#!/usr/bin/env python
"""F1 benchmark: fused NF4 dequant + tcgen05 GEMM over a model's linear weights.

One step = Y_t = X_t . W_t^T for every linear weight W_t of the model (X_t:
[M, K_t] bf16 activations), i.e. the quantized matmuls of one forward pass at
batch M (the paper's batches are 2..64).  Compared with the unfused path
the paper optimizes: nf4_dequantize_batched into a bf16 weight buffer, then
torch.matmul (cuBLAS) per weight.

    python tools/gemm_bench.py --model gemma-3-27b --m 16 --layers 8 --steps 20

Prints one JSON line: fused ms/step, unfused ms/step (dequant + cuBLAS), speedup,
effective HBM GB/s (codes + scales + X + Y bytes) and TFLOP/s of the fused path.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2604_02556_b200 as nf4
    from paper_2604_02556_b200 import weights
    from synth import workloads as wl

    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="gemma-3-27b")
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--splits", type=int, default=0,
                    help="0: stream-K (default); -1: classic grid, makespan split heuristic; >0: classic, fixed")
    ap.add_argument("--no-unfused", action="store_true")
    args = ap.parse_args()

    torch.cuda.set_device(0)
    nf4.load()
    tensors = wl.model_tensors(args.model, layers=args.layers)
    ws = weights.from_hash(tensors, 64, True, "bf16", seed0=7, device="cuda")
    M = args.m
    xs = {}
    for t in tensors:
        if t.cols not in xs:
            xs[t.cols] = torch.randn(M, t.cols, device="cuda").to(torch.bfloat16)
    ys = [torch.empty(M, t.rows, dtype=torch.bfloat16, device="cuda") for t in tensors]
    wsp = {}
    dqs = []
    for i, (t, e) in enumerate(zip(tensors, ws.entries)):
        nb = e.n // 64
        dqs.append(nf4.DQ(ws._ptr(ws.scales, e.scale_off), ws.code2.data_ptr(), ws._ptr(ws.groups, e.group_off),
                          e.offset))
    splits = {}
    for t in tensors:
        key = (t.rows, t.cols)
        if key not in splits:
            s = nf4.nf4_gemm_default_splits(M, t.rows, t.cols) if args.splits < 0 else args.splits
            splits[key] = s
            b = nf4.nf4_gemm_workspace_bytes(M, t.rows, t.cols, s)
            wsp[key] = torch.zeros(max(b, 16), dtype=torch.uint8, device="cuda")

    def fused_step():
        for i, (t, e) in enumerate(zip(tensors, ws.entries)):
            key = (t.rows, t.cols)
            nf4.nf4_gemm(xs[t.cols], ws._ptr(ws.codes, e.codes_off), None, dqs[i], N=t.rows, K=t.cols,
                         y=ys[i], splits=splits[key], workspace=wsp[key])

    def timeit(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / args.steps

    fused_ms = timeit(fused_step)
    n_total = sum(t.n for t in tensors)
    bytes_w = sum((e.n // 2) + (e.n // 64) + 4 * (e.n // 64 // 256) for e in ws.entries)
    bytes_xy = sum(M * t.cols * 2 + M * t.rows * 2 for t in tensors)
    flops = 2.0 * M * n_total
    res = {"model": args.model, "layers": args.layers or wl.MODELS[args.model][0], "M": M,
           "tensors": len(tensors), "weight_elements": n_total,
           "fused_ms": round(fused_ms, 4),
           "fused_hbm_gbs": round((bytes_w + bytes_xy) / (fused_ms * 1e-3) / 1e9, 1),
           "fused_tflops": round(flops / (fused_ms * 1e-3) / 1e12, 2),
           "splits": sorted(set(splits.values()))}
    if not args.no_unfused:
        wbuf = torch.empty(max(t.n for t in tensors), dtype=torch.bfloat16, device="cuda")

        def unfused_step():
            for i, (t, e) in enumerate(zip(tensors, ws.entries)):
                nf4.nf4_dequantize(ws._ptr(ws.codes, e.codes_off), None, dqs[i], n=e.n, blocksize=64,
                                   out_dtype="bf16", out=wbuf)
                torch.matmul(xs[t.cols], wbuf[:e.n].view(t.rows, t.cols).t(), out=ys[i])

        unfused_ms = timeit(unfused_step)
        res["unfused_ms"] = round(unfused_ms, 4)
        res["speedup_vs_unfused"] = round(unfused_ms / fused_ms, 3)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
