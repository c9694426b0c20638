#!/usr/bin/env python
"""dequantizing ONE decoder layer (7 projections), the unit the
paper's inference loop invokes per layer.  Compares 7 single-tensor
launches, one nf4_dequantize_batched launch, and that launch replayed from a
CUDA graph.  CUDA events, median of --reps.

    python tools/layer_latency.py --model gemma-3-27b
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
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
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    tensors = wl.model_tensors(args.model, layers=1)
    ws = stores.from_hash(tensors, 64, True, "bf16", seed0=11, device="cuda")
    descs = ws.nf4_tensors()
    s = torch.cuda.Stream()
    flush = torch.ones(512 << 20, dtype=torch.uint8, device="cuda")
    sink = torch.empty(1, dtype=torch.int64, device="cuda")

    def separate():
        for d in descs:
            nf4.nf4_dequantize_batched([d], "bf16", stream=s)

    def batched():
        nf4.nf4_dequantize_batched(descs, "bf16", stream=s)

    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        batched()

    def time_it(fn, cold, mean=False):
        ts = []
        for r in range(args.reps + 3):
            with torch.cuda.stream(s):
                if cold:
                    sink.copy_(flush.sum(dtype=torch.int64))
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                fn()
                b.record(s)
            s.synchronize()
            if r >= 3:
                ts.append(a.elapsed_time(b) * 1e3)
        return statistics.mean(ts) if mean else statistics.median(ts)

    alg = ws.algorithmic_bytes()
    res = {"model": args.model, "tensors": len(tensors), "elements": ws.n_total, "algorithmic_bytes": alg}
    for name, fn in (("7_launches", separate), ("batched_1_launch", batched), ("cuda_graph", g.replay)):
        for cold in (True, False):
            us = time_it(fn, cold)
            res[f"{name}_{'cold' if cold else 'hot'}_us"] = round(us, 1)
            res[f"{name}_{'cold' if cold else 'hot'}_gbs"] = round(alg / (us * 1e-6) / 1e9, 1)
    # each projection as its own tensor: one launch, cold.  Single
    # cold launches are this short that the event timestamps' ~2 us granularity shows in
    # every sample, so these are MEANS over the reps (medians land on multiples of 2.048 us).
    per = []
    for t, d, e in zip(tensors, descs, ws.entries):
        nb = -(-e.n // 64)
        tb = (e.n + 1) // 2 + 2 * e.n + nb + 4 * (-(-nb // 256))
        us = time_it(lambda d=d: nf4.nf4_dequantize_batched([d], "bf16", stream=s), True, mean=True)
        per.append({"tensor": t.name, "shape": [t.rows, t.cols], "elements": e.n, "cold_us_mean": round(us, 2),
                    "cold_gbs": round(tb / (us * 1e-6) / 1e9, 1)})
    res["per_tensor"] = per
    # floor of this measurement: a trivial one-block kernel timed the same way
    res["trivial_kernel_cold_us_mean"] = round(time_it(lambda: sink.zero_(), True, mean=True), 2)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
