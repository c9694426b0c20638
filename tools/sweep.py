#!/usr/bin/env python
"""BASELINE config 5 sweep: blocksize 64/128/256/4096 x fp16/bf16 x n = 2^20..2^30
(fp32 absmax primary; --dq for double-quant), 1 GPU, single-tensor nf4_dequantize.

Default method "graph": every point is K launches replayed from one CUDA graph
(back to back, as a stream of weight dequantizations runs), time per launch =
graph time / K.  Points whose footprint fits in ~4x L2 rotate over R disjoint
copies of inputs and outputs (R x footprint > 4 x L2), so every launch is
L2-cold.  Method "events" (round 1): CUDA events around single launches with a
512 MB read flush before each cold one -- it carries a ~6 us event/launch floor.
Prints a markdown table and writes JSON lines to --out.
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
    from paper_2604_02556_b200 import _lib
    from synth import workloads as wl

    ap = argparse.ArgumentParser()
    ap.add_argument("--dq", action="store_true")
    ap.add_argument("--min-log2", type=int, default=20)
    ap.add_argument("--max-log2", type=int, default=30)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    ap.add_argument("--method", default="graph", choices=["graph", "events"])
    ap.add_argument("--launches", type=int, default=64, help="graph method: launches per replay")
    ap.add_argument("--early-inputs", action="store_true", help="nf4_set_early_input_reads(1)")
    ap.add_argument("--bs", default="64,128,256,4096")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    nf4.load()
    if args.early_inputs:
        nf4.nf4_set_early_input_reads(True)
    # L2 flush by READING 512 MB (a write-based flush leaves 256 MB of dirty lines whose
    # lazy write-back would then be charged to the timed launch)
    flush = torch.ones(512 << 20, dtype=torch.uint8, device="cuda")
    sink = torch.empty(1, dtype=torch.int64, device="cuda")
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    nmax = 1 << args.max_log2
    packed = torch.empty(nmax // 2, dtype=torch.uint8, device="cuda")
    nf4.nf4_synth_fill(_lib.NF4_SYNTH_CODES, 5, 0, nmax // 2, packed)
    out = torch.empty(nmax, dtype=torch.int16, device="cuda")
    rows = []
    print("| bs | dtype | n | cold/hot | us | GB/s | % of measured copy | Gelem/s |")
    print("|---|---|---|---|---|---|---|---|")
    for bs in (int(b) for b in args.bs.split(",")):
        nb = nmax // bs
        if args.dq:
            q = torch.empty(nb, dtype=torch.uint8, device="cuda")
            nf4.nf4_synth_fill(_lib.NF4_SYNTH_QABSMAX, 6, 0, nb, q)
            a2 = torch.empty(-(-nb // 256), dtype=torch.float32, device="cuda")
            nf4.nf4_synth_fill(_lib.NF4_SYNTH_ABSMAX2, 6, 0, a2.numel(), a2)
            from synth import inputs as syn
            code2 = torch.from_numpy(syn.dynamic_map_code2()).cuda()
            dq = True
            absmax = None
        else:
            absmax = torch.empty(nb, dtype=torch.float32, device="cuda")
            nf4.nf4_synth_fill(_lib.NF4_SYNTH_ABSMAX, 6, 0, nb, absmax)
            dq = None
        for dt in ("f16", "bf16"):
            for lg in range(args.min_log2, args.max_log2 + 1):
                n = 1 << lg
                cold = n * 2.5 < 4 * 126e6
                reps = 1
                if args.method == "graph":
                    reps = max(1, min(nmax // n, -(-int(4 * 126e6) // int(n * 2.5)))) if cold else 1

                def f(r=0, stream=None):
                    # copy r: elements [r*n, (r+1)*n) of the big buffers (disjoint, 256-B aligned)
                    k0 = r * n
                    if dq is not None:
                        d = nf4.DQ(q[k0 // bs:(k0 + n) // bs], code2, a2[k0 // bs // 256:], 0.05)
                        a = None
                    else:
                        d, a = None, absmax[k0 // bs:(k0 + n) // bs]
                    nf4.nf4_dequantize(packed[k0 // 2:(k0 + n) // 2], a, d, n=n, blocksize=bs, out_dtype=dt,
                                       out=out[k0:k0 + n], stream=stream)
                for r in range(max(3, reps)):
                    f(r % reps)
                torch.cuda.synchronize()
                if args.method == "graph":
                    K = args.launches
                    gs = torch.cuda.Stream()
                    gs.wait_stream(torch.cuda.current_stream())
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=gs):
                        for i in range(K):
                            f(i % reps, gs)
                    g.replay()
                    torch.cuda.synchronize()
                    times = []
                    for _ in range(max(3, args.reps // 4)):
                        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        s.record()
                        g.replay()
                        e.record()
                        torch.cuda.synchronize()
                        times.append(s.elapsed_time(e) / K)
                    del g
                else:
                    times = []
                    for _ in range(args.reps):
                        if cold:
                            sink.copy_(flush.sum(dtype=torch.int64))
                        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        s.record()
                        f()
                        e.record()
                        torch.cuda.synchronize()
                        times.append(s.elapsed_time(e))
                times.sort()
                ms = times[len(times) // 2]
                alg = n * wl.algorithmic_bytes_per_element(bs, args.dq)
                gbs = alg / (ms * 1e-3) / 1e9
                r = {"blocksize": bs, "dtype": dt, "n": n, "dq": args.dq, "cold": cold, "method": args.method,
                     "rotating_copies": reps, "us": round(ms * 1e3, 2),
                     "gbs": round(gbs, 1), "frac_measured_copy": round(gbs / peak, 4),
                     "gelem_s": round(n / (ms * 1e-3) / 1e9, 1)}
                rows.append(r)
                print(f"| {bs} | {dt} | 2^{lg} | {'cold' if cold else 'hot'} | {r['us']} | {r['gbs']} | "
                      f"{100 * r['frac_measured_copy']:.1f}% | {r['gelem_s']} |", flush=True)
    if args.out:
        with open(args.out, "w") as fo:
            for r in rows:
                fo.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
