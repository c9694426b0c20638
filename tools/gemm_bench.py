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
    from synth import stores
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
    ap.add_argument("--graph", action="store_true", help="replay each step from a CUDA graph")
    ap.add_argument("--grouped", action="store_true",
                    help="q/k/v and gate/up of each layer as one nf4_gemm_grouped launch (they share X)")
    ap.add_argument("--multi", action="store_true",
                    help="all weights of the step as independent problems, nf4_gemm_multi (<= 64 per launch)")
    args = ap.parse_args()

    torch.cuda.set_device(0)
    nf4.load()
    tensors = wl.model_tensors(args.model, layers=args.layers)
    ws = stores.from_hash(tensors, 64, True, "bf16", seed0=7, device="cuda")
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

    # groups of consecutive weights sharing X: (q, k, v), (o), (gate, up), (down) per layer
    groups = []
    cur = []
    for i, t in enumerate(tensors):
        kind = t.name.split(".")[2].split("[")[0]
        key = {"q_proj": "qkv", "k_proj": "qkv", "v_proj": "qkv", "gate_proj": "gu", "up_proj": "gu"}.get(kind, kind)
        lay = t.name.split(".")[1]
        if cur and (cur[0][1] != (lay, key) or key not in ("qkv", "gu")):
            groups.append([c[0] for c in cur])
            cur = []
        cur.append((i, (lay, key)))
    if cur:
        groups.append([c[0] for c in cur])
    gws = {}
    for grp in groups:
        if len(grp) > 1:
            Ns = tuple(tensors[i].rows for i in grp)
            K = tensors[grp[0]].cols
            gws[tuple(grp)] = torch.zeros(max(16, nf4.nf4_gemm_grouped_workspace_bytes(M, Ns, K)),
                                          dtype=torch.uint8, device="cuda")

    def grouped_step():
        for grp in groups:
            if len(grp) == 1:
                i = grp[0]
                t, e = tensors[i], ws.entries[i]
                key = (t.rows, t.cols)
                nf4.nf4_gemm(xs[t.cols], ws._ptr(ws.codes, e.codes_off), None, dqs[i], N=t.rows, K=t.cols,
                             y=ys[i], splits=splits[key], workspace=wsp[key])
            else:
                K = tensors[grp[0]].cols
                members = [(ws._ptr(ws.codes, ws.entries[i].codes_off), None, dqs[i], tensors[i].rows) for i in grp]
                nf4.nf4_gemm_grouped(xs[K], members, K=K, ys=[ys[i] for i in grp], workspace=gws[tuple(grp)])

    mws = torch.zeros(max(16, max(nf4.nf4_gemm_multi_workspace_bytes(M, [t.rows for t in tensors[i:i + 64]],
                                                                      [t.cols for t in tensors[i:i + 64]])
                                  for i in range(0, len(tensors), 64))), dtype=torch.uint8, device="cuda")
    probs = [(xs[t.cols], t.cols, ws._ptr(ws.codes, e.codes_off), None, dqs[i], t.rows)
             for i, (t, e) in enumerate(zip(tensors, ws.entries))]

    def multi_step():
        for i in range(0, len(probs), 64):
            nf4.nf4_gemm_multi(probs[i:i + 64], M=M, ys=ys[i:i + 64], workspace=mws)

    step = multi_step if args.multi else grouped_step if args.grouped else fused_step
    if args.graph:
        # the whole step as one CUDA graph (no host launch overhead; PDL edges kept)
        gs = torch.cuda.Stream()
        gs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(gs):
            step()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            step()
        step = graph.replay
    fused_ms = timeit(step)
    n_total = sum(t.n for t in tensors)
    bytes_w = sum((e.n // 2) + (e.n // 64) + 4 * (e.n // 64 // 256) for e in ws.entries)
    bytes_xy = sum(M * t.cols * 2 + M * t.rows * 2 for t in tensors)
    flops = 2.0 * M * n_total
    res = {"model": args.model, "layers": args.layers or wl.MODELS[args.model][0], "M": M,
           "tensors": len(tensors), "weight_elements": n_total,
           "fused_ms": round(fused_ms, 4), "graph": bool(args.graph),
           "fused_hbm_gbs": round((bytes_w + bytes_xy) / (fused_ms * 1e-3) / 1e9, 1),
           "fused_tflops": round(flops / (fused_ms * 1e-3) / 1e12, 2),
           # roofline of the fused kernel: one shared-memory LUT lookup per weight,
           # 6.48 T lookups/s measured on this GPU (profiles/r01_lutbench.txt)
           "fused_tweights_per_s": round(n_total / (fused_ms * 1e-3) / 1e12, 3),
           "frac_of_lut_bound": round(n_total / (fused_ms * 1e-3) / 6.48e12, 3),
           "splits": sorted(set(splits.values())), "grouped": bool(args.grouped),
           "multi": bool(args.multi),
           "launches_per_step": -(-len(tensors) // 64) if args.multi else len(groups) if args.grouped else len(tensors)}
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
