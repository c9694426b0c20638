#!/usr/bin/env python
"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every kernel of libnf4 on tiny, ragged and unaligned inputs.  Exits non-zero on a
parity mismatch so the sanitizer run also checks results.

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_case.py
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import oracle
    import paper_2604_02556_b200 as nf4
    from paper_2604_02556_b200 import _lib
    from synth import inputs as syn

    torch.cuda.set_device(0)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    bad = 0
    code2 = syn.dynamic_map_code2()
    variants = nf4.nf4_kernel_variants()
    only_default = os.environ.get("NF4_SANITIZE_DEFAULT_ONLY") == "1"
    default_v = nf4.nf4_get_kernel_variant()
    passes = [(v, False) for v in ([default_v] if only_default else range(len(variants)))] + [(default_v, True)]
    for v, early in passes:     # the last pass: early input reads (nf4_set_early_input_reads)
        nf4.nf4_set_kernel_variant(v)
        torch.cuda.synchronize()
        nf4.nf4_set_early_input_reads(early)
        for n in (1, 31, 16384 + 77, 3 * 16384):
            for dq in (False, True):
                nb = -(-n // 64)
                packed = syn.hash_packed(n, 0, (n + 1) // 2)
                if dq:
                    kw = dict(qabsmax=syn.hash_qabsmax(n, 0, nb), code2=code2,
                              absmax2=syn.hash_absmax2(n, 0, -(-nb // 256)), offset=float(syn.hash_offset(n)))
                    out = nf4.nf4_dequantize(d(packed), None, nf4.DQ(d(kw["qabsmax"]), d(code2), d(kw["absmax2"]),
                                                                   kw["offset"]), n=n, blocksize=64, out_dtype="bf16")
                else:
                    kw = dict(absmax=syn.hash_absmax(n, 0, nb))
                    out = nf4.nf4_dequantize(d(packed), d(kw["absmax"]), None, n=n, blocksize=64, out_dtype="bf16")
                torch.cuda.synchronize()
                ref = oracle.dequantize(packed, n, 64, oracle.OUT_BF16, **kw)
                bad += int(not np.array_equal(out.view(torch.int16).cpu().numpy().view(np.uint16), ref))
    nf4.nf4_set_early_input_reads(False)
    nf4.nf4_set_kernel_variant(default_v)
    # unaligned output
    n = 5000
    packed = syn.hash_packed(3, 0, n // 2)
    am = syn.hash_absmax(3, 0, -(-n // 64))
    buf = torch.zeros(n + 8, dtype=torch.int16, device="cuda")
    nf4.nf4_dequantize(d(packed), d(am), None, n=n, blocksize=64, out_dtype="f16", out=buf[1:1 + n].view(torch.float16))
    # quantizers
    w = syn.gaussian_weights(4097, 1)
    p, a = nf4.nf4_quantize(d(w), 64)
    q = nf4.nf4_double_quantize(a, 0.05, d(code2))
    # fused GEMM (both split modes), tiny
    x = torch.randn(3, 256, device="cuda").to(torch.bfloat16)
    wp = d(syn.hash_packed(9, 0, 128 * 256 // 2))
    wa = d(syn.hash_absmax(9, 0, 128 * 256 // 64))
    for s in (1, 2, 0):
        nf4.nf4_gemm(x, wp, wa, None, N=128, K=256, splits=s)
    # stream-K with tiles cut into several pieces (fix-up path), DQ scales, checked vs the oracle
    M2, N2, K2 = 20, 2048, 1024
    x2 = syn.gaussian_weights(M2 * K2, 2).reshape(M2, K2)
    import ml_dtypes
    x2_16 = x2.astype(ml_dtypes.bfloat16).view(np.uint16)
    wp2 = syn.hash_packed(10, 0, N2 * K2 // 2)
    nb2 = N2 * K2 // 64
    kw2 = dict(qabsmax=syn.hash_qabsmax(10, 0, nb2), code2=code2, absmax2=syn.hash_absmax2(10, 0, -(-nb2 // 256)),
               offset=float(syn.hash_offset(10)))
    xt = d(x2_16.view(np.int16)).view(torch.bfloat16)
    dqt = nf4.DQ(d(kw2["qabsmax"]), d(code2), d(kw2["absmax2"]), kw2["offset"])
    ws2 = torch.zeros(max(16, nf4.nf4_gemm_workspace_bytes(M2, N2, K2, 0)), dtype=torch.uint8, device="cuda")
    for _ in range(2):   # the second call reuses the (self-cleaning) workspace
        y2 = nf4.nf4_gemm(xt, d(wp2), None, dqt, N=N2, K=K2, y_dtype="f32", workspace=ws2)
    torch.cuda.synchronize()
    ref2, mag2 = oracle.gemm_reference(x2_16, oracle.OUT_BF16, wp2, N2, K2, 64, **kw2)
    bad += int(not (np.abs(y2.cpu().numpy().astype(np.float64) - ref2) <= K2 * 2.0 ** -23 * mag2 + 1e-30).all())
    # grouped GEMM (2 members) at three token-tile widths, launched back to back (programmatic
    # dependent launch: the weights are read before griddepcontrol.wait); bit-identical to
    # the single-weight launches
    wp3 = d(syn.hash_packed(11, 0, 256 * 256 // 2))
    wa3 = d(syn.hash_absmax(11, 0, 256 * 256 // 64))
    for Mg in (5, 100, 200):
        xg = torch.randn(Mg, 256, device="cuda").to(torch.bfloat16)
        for _ in range(2):
            yg = nf4.nf4_gemm_grouped(xg, [(wp, wa, None, 128), (wp3, wa3, None, 256)], K=256, y_dtype="f32")
        y0 = nf4.nf4_gemm(xg, wp, wa, None, N=128, K=256, y_dtype="f32")
        y1 = nf4.nf4_gemm(xg, wp3, wa3, None, N=256, K=256, y_dtype="f32")
        torch.cuda.synchronize()
        bad += int(not (torch.equal(yg[0], y0) and torch.equal(yg[1], y1)))
    # multi-problem GEMM (own X and K per problem, mixed scale formats, tiles cut into
    # pieces), launched twice back to back on one workspace; checked vs the oracle bound
    shapes = [(384, 512, True), (200, 1024, False), (256, 256, True)]
    probs, refs = [], []
    for i, (Nm, Km, dqm) in enumerate(shapes):
        pk = syn.hash_packed(20 + i, 0, Nm * Km // 2)
        nbm = Nm * Km // 64
        if dqm:
            kwm = dict(qabsmax=syn.hash_qabsmax(20 + i, 0, nbm), code2=code2,
                       absmax2=syn.hash_absmax2(20 + i, 0, -(-nbm // 256)), offset=float(syn.hash_offset(20 + i)))
        else:
            kwm = dict(absmax=syn.hash_absmax(20 + i, 0, nbm))
        xm = syn.gaussian_weights(24 * Km, 30 + i).reshape(24, Km).astype(ml_dtypes.bfloat16).view(np.uint16)
        xmt = d(xm.view(np.int16)).view(torch.bfloat16)
        dqm_t = nf4.DQ(d(kwm["qabsmax"]), d(code2), d(kwm["absmax2"]), kwm["offset"]) if dqm else None
        probs.append((xmt, Km, d(pk), None if dqm else d(kwm["absmax"]), dqm_t, Nm))
        refs.append(oracle.gemm_reference(xm, oracle.OUT_BF16, pk, Nm, Km, 64, **kwm))
    wsm = torch.zeros(max(16, nf4.nf4_gemm_multi_workspace_bytes(24, [s_[0] for s_ in shapes],
                                                                 [s_[1] for s_ in shapes])),
                      dtype=torch.uint8, device="cuda")
    for _ in range(2):
        ym = nf4.nf4_gemm_multi(probs, M=24, y_dtype="f32", workspace=wsm)
    torch.cuda.synchronize()
    for (Nm, Km, _), yi, (rf, mg) in zip(shapes, ym, refs):
        bad += int(not (np.abs(yi.cpu().numpy().astype(np.float64) - rf) <= Km * 2.0 ** -23 * mg + 1e-30).all())
    # short segments: K = 128 (one super-stage per tile) and several tiles per CTA, so
    # accumulators are reused while earlier segments are in flight (round-2 barrier fix)
    Ns, Ks = 128 * 148 * 2 + 64, 128
    pks = syn.hash_packed(40, 0, Ns * Ks // 2)
    ams = syn.hash_absmax(40, 0, Ns * Ks // 64)
    xs16 = syn.gaussian_weights(16 * Ks, 41).reshape(16, Ks).astype(ml_dtypes.bfloat16).view(np.uint16)
    xst = d(xs16.view(np.int16)).view(torch.bfloat16)
    for _ in range(2):
        ys_ = nf4.nf4_gemm(xst, d(pks), d(ams), None, N=Ns, K=Ks, y_dtype="f32")
    torch.cuda.synchronize()
    rfs, mgs = oracle.gemm_reference(xs16, oracle.OUT_BF16, pks, Ns, Ks, 64, absmax=ams)
    bad += int(not (np.abs(ys_.cpu().numpy().astype(np.float64) - rfs) <= Ks * 2.0 ** -23 * mgs + 1e-30).all())
    # synth + sol
    buf8 = torch.empty(8192 * 4, dtype=torch.uint8, device="cuda")
    nf4.nf4_synth_fill(_lib.NF4_SYNTH_CODES, 1, 3, 1000, buf8)
    nf4.nf4_synth_fill(_lib.NF4_SYNTH_CODES, 1, 0, buf8.numel(), buf8)
    dst = torch.empty(8192 * 16, dtype=torch.uint8, device="cuda")
    nf4.nf4_sol_stream(buf8, 8192 * 4, dst)
    torch.cuda.synchronize()
    print("sanitize_case: parity mismatches =", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
