"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, bit-exact
(0 ULP, every 16-bit output word; NaN class only -- reading R9).

Inputs come from synth/ (host numpy) or from the oracle quantizer, never from
the CUDA path; expected values come only from oracle/.  Sizes span several
16384-element tiles plus ragged tails; the full-size test uses the bench's own
launch configuration (WeightStore.dequantize_all) on sampled blocks.
"""
from __future__ import annotations

import numpy as np
import pytest

from synth import inputs as syn
from synth import workloads as wl
from tests import npref

pytestmark = pytest.mark.gpu

TILE = 16384


@pytest.fixture(scope="module")
def nf4():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_02556_b200 as m
    m.load()
    m.nf4_set_max_ctas(0)
    return m


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host16(t):
    import torch
    torch.cuda.synchronize()
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def _inputs(n, bs, dq, seed):
    nb = -(-n // bs)
    packed = syn.hash_packed(seed, 0, (n + 1) // 2)
    if dq:
        return packed, dict(qabsmax=syn.hash_qabsmax(seed, 0, nb), code2=syn.dynamic_map_code2(),
                            absmax2=syn.hash_absmax2(seed, 0, -(-nb // 256)), offset=float(syn.hash_offset(seed)))
    return packed, dict(absmax=syn.hash_absmax(seed, 0, nb))


def _gpu_deq(nf4, packed, kw, n, bs, dtype, out=None):
    if "absmax" in kw:
        return nf4.nf4_dequantize(dev(packed), dev(kw["absmax"]), None, n=n, blocksize=bs, out_dtype=dtype, out=out)
    dq = nf4.DQ(dev(kw["qabsmax"]), dev(kw["code2"]), dev(kw["absmax2"]), kw["offset"])
    return nf4.nf4_dequantize(dev(packed), None, dq, n=n, blocksize=bs, out_dtype=dtype, out=out)


def _oracle(orc, packed, kw, n, bs, dtype, threads=8):
    return orc.dequantize(packed, n, bs, orc.OUT_F16 if dtype == "f16" else orc.OUT_BF16, threads=threads, **kw)


SIZES = [1, 2, 3, 15, 16, 17, 63, 64, 65, 127, 1023, 1024, 1025, TILE - 1, TILE, TILE + 1,
         3 * TILE + 777, 5 * TILE + 16 * 37, 257 * 64 * 3 + 5]


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("dq", [False, True])
@pytest.mark.parametrize("bs", [64, 128, 256, 4096])
def test_parity_sizes_blocksizes(nf4, orc, dtype, dq, bs):
    for n in SIZES:
        packed, kw = _inputs(n, bs, dq, seed=n + bs)
        got = host16(_gpu_deq(nf4, packed, kw, n, bs, dtype))
        ref = _oracle(orc, packed, kw, n, bs, dtype)
        bad = ~npref.same_bits(got, ref, dtype)
        assert not bad.any(), (n, bs, np.nonzero(bad)[0][:5])


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_parity_realistic_gaussian_qlora(nf4, orc, dtype):
    """Gaussian weights -> oracle quantize + double quantize (realistic code and
    scale distributions) -> GPU vs oracle."""
    n, bs = 4096 * 1024 + 4096, 64
    w = syn.gaussian_weights(n, 123)
    packed, absmax = orc.quantize(w, bs)
    code2 = syn.dynamic_map_code2()
    off = float(np.float32(absmax.astype(np.float64).mean()))
    q, a2 = orc.double_quantize(absmax, off, code2)
    for kw in (dict(absmax=absmax), dict(qabsmax=q, code2=code2, absmax2=a2, offset=off)):
        got = host16(_gpu_deq(nf4, packed, kw, n, bs, dtype))
        ref = _oracle(orc, packed, kw, n, bs, dtype)
        assert np.array_equal(got, ref)


def test_parity_special_values(nf4, orc):
    """Signed zeros, subnormal and huge absmax, fp16 overflow to Inf, NaN/Inf
    absmax (NaN compared by class), all 256 bytes (S:203 scale set)."""
    packed = np.tile(np.arange(256, dtype=np.uint8), 64)           # 16384 bytes = 32768 elements
    n = packed.size * 2
    specials = np.array([0.0, -0.0, 1.0, 0.5, 3.14159e-3, 6.5504e4, 1e-39, 1e-45, 3.0e38, np.inf, np.nan,
                         65520.0, 1e5, 2.0 ** -24, 7.0, 1e-8], np.float32)
    absmax = np.resize(specials, n // 64)
    for dtype in ("f16", "bf16"):
        got = host16(_gpu_deq(nf4, packed, dict(absmax=absmax), n, 64, dtype))
        ref = _oracle(orc, packed, dict(absmax=absmax), n, 64, dtype)
        assert npref.same_bits(got, ref, dtype).all()


@pytest.mark.parametrize("dq", [False, True])
def test_all_kernel_variants_bit_exact(nf4, orc, dq):
    """Every dequant variant (vector width, unroll, persistent or one CTA per
    tile) gives the oracle's bytes, including tails and small tensors."""
    names = nf4.nf4_kernel_variants()
    default = nf4.nf4_get_kernel_variant()
    try:
        for v in range(len(names)):
            assert nf4.nf4_set_kernel_variant(v) == v
            for dtype in ("f16", "bf16"):
                for n in (1, 33, 1025, 2 * TILE - 7, 5 * TILE, 9 * TILE + 4099):
                    packed, kw = _inputs(n, 64, dq, 3 * n + v)
                    got = host16(_gpu_deq(nf4, packed, kw, n, 64, dtype))
                    assert np.array_equal(got, _oracle(orc, packed, kw, n, 64, dtype)), (names[v], dtype, n)
    finally:
        nf4.nf4_set_kernel_variant(default)


def test_grid_size_invariance(nf4, orc):
    """Identical bytes for 1 CTA, one wave, and the automatic persistent grid."""
    import torch
    n, bs = 37 * TILE + 999, 64
    packed, kw = _inputs(n, bs, True, 77)
    outs = []
    for cap in (1, 7, 148, 0):
        nf4.nf4_set_max_ctas(cap)
        outs.append(host16(_gpu_deq(nf4, packed, kw, n, bs, "bf16")))
    nf4.nf4_set_max_ctas(0)
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    assert np.array_equal(outs[0], _oracle(orc, packed, kw, n, bs, "bf16"))
    assert nf4.nf4_dequant_grid(10 ** 9) >= torch.cuda.get_device_properties(0).multi_processor_count


@pytest.mark.parametrize("dq", [False, True])
def test_unaligned_buffers_and_canary(nf4, orc, dq):
    """Any alignment of packed/out is exact (element path) and nothing past
    out[n-1] is written."""
    import torch
    n, bs = 2 * TILE + 333, 64
    packed, kw = _inputs(n, bs, dq, 5)
    ref = _oracle(orc, packed, kw, n, bs, "f16")
    for pk_off, out_off in ((1, 0), (0, 1), (3, 5), (8, 16)):
        pbuf = torch.zeros(packed.size + 16, dtype=torch.uint8, device="cuda")
        pbuf[pk_off:pk_off + packed.size] = dev(packed)
        obuf = torch.full((n + 64,), 0x5A5A, dtype=torch.int16, device="cuda")
        out = obuf[out_off:out_off + n].view(torch.float16)
        if dq:
            d = nf4.DQ(dev(kw["qabsmax"]), dev(kw["code2"]), dev(kw["absmax2"]), kw["offset"])
            nf4.nf4_dequantize(pbuf[pk_off:], None, d, n=n, blocksize=bs, out_dtype="f16", out=out)
        else:
            nf4.nf4_dequantize(pbuf[pk_off:], dev(kw["absmax"]), None, n=n, blocksize=bs, out_dtype="f16", out=out)
        full = host16(obuf)
        assert np.array_equal(full[out_off:out_off + n], ref)
        assert (full[:out_off] == 0x5A5A).all() and (full[out_off + n:] == 0x5A5A).all()


def test_batched_mixed_many_tensors(nf4, orc):
    """> NF4_MAX_BATCH tensors (split into several launches), mixed fp32/DQ
    modes, block sizes and ragged sizes, empty tensors included."""
    import torch
    rng = np.random.Generator(np.random.Philox(1))
    specs, descs, refs, outs = [], [], [], []
    for i in range(300):
        n = int(rng.integers(0, 3 * TILE)) if i % 17 else 0
        bs = int([64, 128, 256, 4096][i % 4])
        dq = bool(i % 3 == 0)
        packed, kw = _inputs(n, bs, dq, 1000 + i)
        out = torch.empty(max(n, 1), dtype=torch.float16, device="cuda")
        t = dict(packed=dev(packed) if n else None, out=out)
        if dq:
            t["dq"] = nf4.DQ(dev(kw["qabsmax"]), dev(kw["code2"]), dev(kw["absmax2"]), kw["offset"])
        else:
            t["absmax"] = dev(kw["absmax"])
        specs.append(t)
        descs.append(nf4.NF4Tensor(t["packed"], n, bs, out, t.get("absmax"), t.get("dq")))
        refs.append(_oracle(orc, packed, kw, n, bs, "f16") if n else None)
        outs.append((out, n))
    nf4.nf4_dequantize_batched(descs, "f16")
    assert nf4.nf4_last_launch_count() == -(-sum(1 for d in descs if d.n) // 128)
    for (out, n), ref in zip(outs, refs):
        if n:
            assert np.array_equal(host16(out)[:n], ref)


def test_non_default_stream(nf4, orc):
    import torch
    n, bs = 9 * TILE, 64
    packed, kw = _inputs(n, bs, False, 9)
    s = torch.cuda.Stream()
    p, a = dev(packed), dev(kw["absmax"])
    out = torch.empty(n, dtype=torch.float16, device="cuda")
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        nf4.nf4_dequantize(p, a, None, n=n, blocksize=bs, out_dtype="f16", out=out, stream=s)
    s.synchronize()
    assert np.array_equal(host16(out), _oracle(orc, packed, kw, n, bs, "f16"))


def test_error_codes_on_device(nf4):
    import torch
    p = torch.zeros(64, dtype=torch.uint8, device="cuda")
    a = torch.ones(2, dtype=torch.float32, device="cuda")
    o = torch.empty(128, dtype=torch.float16, device="cuda")
    with pytest.raises(nf4.NF4Error) as e:
        nf4.nf4_dequantize(p, a, None, n=128, blocksize=100, out_dtype="f16", out=o)
    assert e.value.status == 3
    with pytest.raises(nf4.NF4Error) as e:
        nf4.nf4_dequantize(p, a.view(torch.uint8)[1:].data_ptr(), None, n=128, blocksize=64,
                           out_dtype="f16", out=o)
    assert e.value.status == 5


# ---------------------------------------------------------------------------
# quantizer (F2): GPU nf4_quantize / nf4_double_quantize == oracle quantizer
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("bs", [64, 128, 256, 4096])
def test_quantize_parity(nf4, orc, bs):
    import torch
    for n in (1, 63, 64, 65, 1000, 64 * 1024 + 31, 300000):
        w = syn.gaussian_weights(n, n + bs)
        w[:: max(1, n // 7)] *= np.float32(-3.0)
        if n > 200:
            w[64:128] = 0.0                                  # an all-zero block
        ref_p, ref_a = orc.quantize(w, bs)
        p, a = nf4.nf4_quantize(dev(w), bs)
        torch.cuda.synchronize()
        assert np.array_equal(p.cpu().numpy(), ref_p), n
        assert np.array_equal(a.cpu().numpy().view(np.uint32), ref_a.view(np.uint32)), n
        # bf16 / fp16 inputs are converted exactly to fp32
        for tdt, npdt in ((torch.float16, np.float16), (torch.bfloat16, None)):
            wt = dev(w).to(tdt)
            w32 = wt.float().cpu().numpy()
            rp, ra = orc.quantize(w32, bs)
            p2, a2 = nf4.nf4_quantize(wt, bs)
            torch.cuda.synchronize()
            assert np.array_equal(p2.cpu().numpy(), rp) and np.array_equal(a2.cpu().numpy(), ra)


def test_double_quantize_parity(nf4, orc):
    import torch
    code2 = syn.dynamic_map_code2()
    for nb in (1, 255, 256, 257, 4096 * 3 + 17):
        absmax = syn.hash_absmax(nb, 0, nb)
        absmax[:: 97] = np.float32(0.0625)
        off = float(np.float32(absmax.astype(np.float64).mean()))
        rq, ra2 = orc.double_quantize(absmax, off, code2)
        d = nf4.nf4_double_quantize(dev(absmax), off, dev(code2))
        torch.cuda.synchronize()
        assert np.array_equal(d.qabsmax.cpu().numpy(), rq)
        assert np.array_equal(d.absmax2.cpu().numpy(), ra2)
    # exact ties between adjacent code2 entries go to the lower index
    from tests.test_oracle_pins import dq_tie_fixture
    c2, cases = dq_tie_fixture()
    for absmax, off, exp in cases:
        rq, _ = orc.double_quantize(absmax, off, c2)
        d = nf4.nf4_double_quantize(dev(absmax), off, dev(c2))
        torch.cuda.synchronize()
        got = d.qabsmax.cpu().numpy()
        assert np.array_equal(got, rq)
        assert all(got[b] == i for b, i in exp.items())
        # the brute-force (unsorted-table) path takes the same tie decision
        perm = np.arange(256)[::-1].copy()
        d = nf4.nf4_double_quantize(dev(absmax), off, dev(c2[perm]))
        rq2, _ = orc.double_quantize(absmax, off, c2[perm])
        torch.cuda.synchronize()
        assert np.array_equal(d.qabsmax.cpu().numpy(), rq2)
    # unsorted code2 takes the brute-force path
    perm = np.random.Generator(np.random.Philox(3)).permutation(256)
    c2u = code2[perm]
    absmax = syn.hash_absmax(5, 0, 1000)
    rq, ra2 = orc.double_quantize(absmax, 0.04, c2u)
    d = nf4.nf4_double_quantize(dev(absmax), 0.04, dev(c2u))
    torch.cuda.synchronize()
    assert np.array_equal(d.qabsmax.cpu().numpy(), rq)


# ---------------------------------------------------------------------------
# input generator (same counter-based hash on both sides)
# ---------------------------------------------------------------------------
def test_synth_fill_matches_host_generator(nf4):
    import torch
    from paper_2604_02556_b200 import _lib
    for begin, count in ((0, 1000), (5, 4099), (123456789, 77)):
        buf = torch.empty(count, dtype=torch.uint8, device="cuda")
        nf4.nf4_synth_fill(_lib.NF4_SYNTH_CODES, 42, begin, count, buf)
        torch.cuda.synchronize()
        assert np.array_equal(buf.cpu().numpy(), syn.hash_packed(42, begin, count))
        f = torch.empty(count, dtype=torch.float32, device="cuda")
        nf4.nf4_synth_fill(_lib.NF4_SYNTH_ABSMAX2, 42, begin, count, f)
        torch.cuda.synchronize()
        assert np.array_equal(f.cpu().numpy(), syn.hash_absmax2(42, begin, count))


# ---------------------------------------------------------------------------
# full size, bench launch configuration, sampled blocks
# ---------------------------------------------------------------------------
def _check_store_sampled(ws, orc, blocks_per_tensor=24, seed=0):
    """For sampled blocks of every tensor, regenerate that block's inputs on the
    host (synth) and compare the oracle with the device outputs."""
    import torch
    rng = np.random.Generator(np.random.Philox(seed))
    bs = ws.blocksize
    code2 = syn.dynamic_map_code2()
    torch.cuda.synchronize()
    checked = 0
    for i, e in enumerate(ws.entries):
        nb = -(-e.n // bs)
        picks = set(rng.integers(0, nb, blocks_per_tensor).tolist()) | {0, nb - 1}
        for b in sorted(picks):
            k0, k1 = b * bs, min(e.n, (b + 1) * bs)
            packed = syn.hash_packed(e.seed, k0 // 2, (k1 - k0 + 1) // 2)
            if ws.dq:
                kw = dict(qabsmax=syn.hash_qabsmax(e.seed, b, 1), code2=code2,
                          absmax2=syn.hash_absmax2(e.seed, b // 256, 1), offset=float(syn.hash_offset(e.seed)))
            else:
                kw = dict(absmax=syn.hash_absmax(e.seed, b, 1))
            ref = orc.dequantize(packed, k1 - k0, bs, orc.OUT_F16 if ws.out_dtype == "f16" else orc.OUT_BF16, **kw)
            got = ws.out_words(i, k0, k1).cpu().numpy().view(np.uint16)
            assert np.array_equal(got, ref), (e.name, b)
            checked += 1
    return checked


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_full_size_configs_sampled(nf4, orc, cfg):
    import torch
    from synth import stores
    c = wl.CONFIGS[cfg]
    tensors = wl.config_tensors(cfg)
    ws = stores.from_hash(tensors, c.blocksize, c.dq, c.out_dtype, seed0=1000 * int(cfg[-1]), device="cuda")
    ws.dequantize_all()
    n_checked = _check_store_sampled(ws, orc, blocks_per_tensor=8 if cfg != "cfg1" else 4096)
    assert n_checked > len(tensors)
    if cfg == "cfg1":
        # config 1 fits the oracle in seconds: compare every element
        e = ws.entries[0]
        packed = syn.hash_packed(e.seed, 0, e.n // 2)
        ref = orc.dequantize(packed, e.n, 64, orc.OUT_F16, absmax=syn.hash_absmax(e.seed, 0, e.n // 64), threads=8)
        assert np.array_equal(ws.out_words(0, 0, e.n).cpu().numpy().view(np.uint16), ref)
    del ws
    torch.cuda.empty_cache()


def test_llama_rank_shard_sampled(nf4, orc):
    """Config 4: rank 3 of the 8-way row sharding (each rank dequantizes its own shard)."""
    import torch
    from synth import stores
    tensors = wl.config_tensors("cfg4", world_size=8, rank=3)
    ws = stores.from_hash(tensors, 64, True, "bf16", seed0=4000 + 3 * 100000, device="cuda")
    ws.dequantize_all()
    assert _check_store_sampled(ws, orc, blocks_per_tensor=4) > 0
    del ws
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dq", [False, True])
def test_host_buffer_path(nf4, orc, dq):
    """nf4_dequantize_host (pinned host in, pinned host out) == oracle."""
    import torch
    n, bs = 10 * 256 * 64 + 4099, 64
    packed, kw = _inputs(n, bs, dq, 31)
    ref = _oracle(orc, packed, kw, n, bs, "bf16")
    chunk = 2 * 256 * 64
    ws = torch.empty(nf4.nf4_host_workspace_bytes(chunk, bs, dq), dtype=torch.uint8, device="cuda")
    pk = torch.from_numpy(packed).pin_memory()
    out = torch.empty(n, dtype=torch.int16).pin_memory()
    if dq:
        d = nf4.DQ(torch.from_numpy(kw["qabsmax"]).pin_memory(), torch.from_numpy(kw["code2"]).pin_memory(),
                   torch.from_numpy(kw["absmax2"]).pin_memory(), kw["offset"])
        nf4.nf4_dequantize_host(pk, None, d, n=n, blocksize=bs, out_dtype="bf16", out=out, workspace=ws,
                                chunk_elems=chunk)
    else:
        nf4.nf4_dequantize_host(pk, torch.from_numpy(kw["absmax"]).pin_memory(), None, n=n, blocksize=bs,
                                out_dtype="bf16", out=out, workspace=ws, chunk_elems=chunk)
    assert np.array_equal(out.numpy().view(np.uint16), ref)


def test_sol_stream(nf4):
    import torch
    src = torch.randint(0, 256, (8192 * 37,), dtype=torch.uint8, device="cuda")
    dst = torch.empty(src.numel() * 4, dtype=torch.uint8, device="cuda")
    nf4.nf4_sol_stream(src, src.numel(), dst)
    torch.cuda.synchronize()
    s = src.cpu().numpy().view(np.uint32).astype(np.uint64)
    d = dst.cpu().numpy().view(np.uint32).reshape(-1, 4)
    x = ((s * 0x00010001) & 0xFFFFFFFF).astype(np.uint32)
    assert np.array_equal(d, np.stack([x, x, x, x], 1))


# ---------------------------------------------------------------------------
# other 16-entry codebooks, fp32 output
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", ["f16", "bf16", "f32"])
@pytest.mark.parametrize("book", ["fp4", "custom"])
def test_codebook_ex_parity(nf4, orc, dtype, book):
    import torch
    cb = (np.array(nf4.nf4_codebook_fp4(), np.float32) if book == "fp4"
          else np.random.Generator(np.random.Philox(4)).standard_normal(16).astype(np.float32))
    if book == "fp4":
        assert np.array_equal(cb, syn.bnb_fp4_codebook())
    code = {"f16": orc.OUT_F16, "bf16": orc.OUT_BF16, "f32": orc.OUT_F32}[dtype]
    for dq in (False, True):
        for n in (1, 77, 3 * TILE + 999, 10 * TILE):
            packed, kw = _inputs(n, 64, dq, n * 3 + 1)
            if dq:
                d = nf4.DQ(dev(kw["qabsmax"]), dev(kw["code2"]), dev(kw["absmax2"]), kw["offset"])
                out = nf4.nf4_dequantize_ex(dev(packed), None, d, n=n, blocksize=64, codebook=cb, out_dtype=dtype)
            else:
                out = nf4.nf4_dequantize_ex(dev(packed), dev(kw["absmax"]), None, n=n, blocksize=64, codebook=cb,
                                            out_dtype=dtype)
            torch.cuda.synchronize()
            got = out.view(torch.int32 if dtype == "f32" else torch.int16).cpu().numpy()
            got = got.view(np.uint32 if dtype == "f32" else np.uint16)
            ref = orc.dequantize(packed, n, 64, code, codebook=cb, threads=8, **kw)
            assert np.array_equal(got, ref), (book, dtype, dq, n)


def test_batched_ex_fp32_nf4(nf4, orc):
    import torch
    descs, refs = [], []
    for i, n in enumerate((5 * TILE, 4097, 2 * TILE + 64)):
        packed, kw = _inputs(n, 128, False, 50 + i)
        out = torch.empty(n, dtype=torch.float32, device="cuda")
        descs.append(nf4.NF4Tensor(dev(packed), n, 128, out, dev(kw["absmax"]), None))
        refs.append(orc.dequantize(packed, n, 128, orc.OUT_F32, **kw))
    nf4.nf4_dequantize_batched_ex(descs, None, "f32")
    torch.cuda.synchronize()
    for d, ref in zip(descs, refs):
        assert np.array_equal(d.out.cpu().numpy().view(np.uint32), ref)


def test_batched_dequant_captured_in_cuda_graph(nf4, orc):
    """The batched path is graph-capturable (no host syncs, no allocations): a
    whole 'model' step captured once and replayed gives the oracle's bytes."""
    import torch
    descs, refs = [], []
    for i, n in enumerate((7 * TILE, 3 * TILE + 5, 1000, 12 * TILE)):
        packed, kw = _inputs(n, 64, bool(i % 2), 200 + i)
        out = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
        if "absmax" in kw:
            descs.append(nf4.NF4Tensor(dev(packed), n, 64, out, dev(kw["absmax"]), None))
        else:
            descs.append(nf4.NF4Tensor(dev(packed), n, 64, out, None,
                                       nf4.DQ(dev(kw["qabsmax"]), dev(kw["code2"]), dev(kw["absmax2"]), kw["offset"])))
        refs.append(_oracle(orc, packed, kw, n, 64, "bf16"))
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        nf4.nf4_dequantize_batched(descs, "bf16", stream=s)
    for d in descs:
        d.out.zero_()
    torch.cuda.synchronize()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    for d, ref in zip(descs, refs):
        assert np.array_equal(host16(d.out), ref)


def test_single_tensor_beyond_2_pow_32_elements(nf4, orc):
    """64-bit indexing: one tensor of 2^32 + 4160 elements (ragged tail); sampled
    blocks around 2^31, 2^32 and the tail are checked against the oracle."""
    import torch
    from paper_2604_02556_b200 import _lib
    n = (1 << 32) + 4160
    bs = 64
    nb = -(-n // bs)
    seed = 77
    packed = torch.empty((n + 1) // 2, dtype=torch.uint8, device="cuda")
    nf4.nf4_synth_fill(_lib.NF4_SYNTH_CODES, seed, 0, packed.numel(), packed)
    absmax = torch.empty(nb, dtype=torch.float32, device="cuda")
    nf4.nf4_synth_fill(_lib.NF4_SYNTH_ABSMAX, seed, 0, nb, absmax)
    out = torch.empty(n, dtype=torch.int16, device="cuda")
    nf4.nf4_dequantize(packed, absmax, None, n=n, blocksize=bs, out_dtype="bf16", out=out.view(torch.bfloat16))
    torch.cuda.synchronize()
    for b in (0, (1 << 31) // bs - 1, (1 << 31) // bs, (1 << 32) // bs - 1, (1 << 32) // bs, nb - 2, nb - 1):
        k0, k1 = b * bs, min(n, (b + 1) * bs)
        ref = orc.dequantize(syn.hash_packed(seed, k0 // 2, (k1 - k0 + 1) // 2), k1 - k0, bs, orc.OUT_BF16,
                             absmax=syn.hash_absmax(seed, b, 1))
        assert np.array_equal(out[k0:k1].cpu().numpy().view(np.uint16), ref), b
    del packed, absmax, out
    torch.cuda.empty_cache()


def test_host_buffer_batched_pipeline(nf4, orc):
    """nf4_dequantize_host_batched: ragged tensors of mixed modes and block sizes
    streamed through one triple-buffered pipeline == oracle."""
    import torch
    chunk = 256 * 4096
    specs = [(3 * chunk + 12345, 64, True), (777, 128, False), (chunk, 4096, True), (2 * chunk - 64, 256, False)]
    ws = torch.empty(nf4.nf4_host_workspace_bytes(chunk, 64, True), dtype=torch.uint8, device="cuda")
    descs, refs = [], []
    for i, (n, bs, dq) in enumerate(specs):
        packed, kw = _inputs(n, bs, dq, 900 + i)
        refs.append(_oracle(orc, packed, kw, n, bs, "f16"))
        out = torch.zeros(n, dtype=torch.int16).pin_memory()
        pk = torch.from_numpy(packed).pin_memory()
        if dq:
            d = nf4.DQ(torch.from_numpy(kw["qabsmax"]).pin_memory(), torch.from_numpy(kw["code2"]).pin_memory(),
                       torch.from_numpy(kw["absmax2"]).pin_memory(), kw["offset"])
            descs.append(nf4.NF4Tensor(pk, n, bs, out, None, d))
        else:
            descs.append(nf4.NF4Tensor(pk, n, bs, out, torch.from_numpy(kw["absmax"]).pin_memory(), None))
    nf4.nf4_dequantize_host_batched(descs, "f16", workspace=ws, chunk_elems=chunk)
    for d, ref in zip(descs, refs):
        assert np.array_equal(d.out.numpy().view(np.uint16), ref)


def test_host_buffer_batched_mixed_fp32_and_dq_small_blocks(nf4, orc):
    """an fp32-absmax tensor at blocksize 64 in a batch that also
    holds double-quant tensors (workspace sized for dq) must not spill its
    scale copy into the slot's output region; several chunks per tensor so the
    three slots are reused."""
    import torch
    chunk = 256 * 64 * 4
    specs = [(5 * chunk + 4097, 64, False), (4 * chunk, 64, True), (3 * chunk + 64, 64, False), (2 * chunk, 128, True)]
    ws = torch.empty(nf4.nf4_host_workspace_bytes(chunk, 64, True), dtype=torch.uint8, device="cuda")
    descs, refs = [], []
    for i, (n, bs, dq) in enumerate(specs):
        packed, kw = _inputs(n, bs, dq, 1900 + i)
        refs.append(_oracle(orc, packed, kw, n, bs, "bf16"))
        out = torch.zeros(n, dtype=torch.int16).pin_memory()
        pk = torch.from_numpy(packed).pin_memory()
        if dq:
            d = nf4.DQ(torch.from_numpy(kw["qabsmax"]).pin_memory(), torch.from_numpy(kw["code2"]).pin_memory(),
                       torch.from_numpy(kw["absmax2"]).pin_memory(), kw["offset"])
            descs.append(nf4.NF4Tensor(pk, n, bs, out, None, d))
        else:
            descs.append(nf4.NF4Tensor(pk, n, bs, out, torch.from_numpy(kw["absmax"]).pin_memory(), None))
    for _ in range(2):
        for d in descs:
            d.out.zero_()
        nf4.nf4_dequantize_host_batched(descs, "bf16", workspace=ws, chunk_elems=chunk)
        for d, ref in zip(descs, refs):
            assert np.array_equal(d.out.numpy().view(np.uint16), ref)


def test_quarter_tile_launches(nf4, orc):
    """Launches below 4 waves of default tiles use 4096-element tiles: single
    tensors around the threshold and decoder-layer-sized batches (<= 16 tensors)
    of ragged, mixed-mode, mixed-blocksize tensors give the oracle's bytes."""
    import torch
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    edge = 4 * sm * TILE
    for n in (edge - TILE - 4097, edge - 1, edge, edge + 3 * 4096 + 5, 3 * 4096 + 17):
        packed, kw = _inputs(n, 64, n % 2 == 0, n % 1000)
        got = host16(_gpu_deq(nf4, packed, kw, n, 64, "f16"))
        assert np.array_equal(got, _oracle(orc, packed, kw, n, 64, "f16")), n
    rng = np.random.Generator(np.random.Philox(9))
    descs, refs = [], []
    for i in range(12):
        n = int(rng.integers(1, 40 * 4096))
        bs = int([64, 128, 256, 4096][i % 4])
        dq = bool(i % 3 == 1)
        packed, kw = _inputs(n, bs, dq, 3000 + i)
        out = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
        if dq:
            d = nf4.DQ(dev(kw["qabsmax"]), dev(kw["code2"]), dev(kw["absmax2"]), kw["offset"])
            descs.append(nf4.NF4Tensor(dev(packed), n, bs, out, None, d))
        else:
            descs.append(nf4.NF4Tensor(dev(packed), n, bs, out, dev(kw["absmax"]), None))
        refs.append(_oracle(orc, packed, kw, n, bs, "bf16"))
    nf4.nf4_dequantize_batched(descs, "bf16")
    torch.cuda.synchronize()
    for d, ref in zip(descs, refs):
        assert np.array_equal(host16(d.out), ref)


@pytest.mark.parametrize("dq", [False, True])
def test_early_input_reads_bit_exact(nf4, orc, dq):
    """nf4_set_early_input_reads(1): inputs read before griddepcontrol.wait, stores
    after it.  A chain of PDL launches where each launch's OUTPUT buffer is still
    being written/read by the previous launches (out buffers reused round-robin, a
    zero-fill kernel between) must give the oracle's bytes: the early reads touch
    only inputs, never `out`.  Default sizes, quarter tiles and the element path."""
    import torch
    cases = [(5 * TILE + 77, 64), (3000, 128), (40 * TILE, 64), (2 * TILE, 4096)]
    data = []
    for i, (n, bs) in enumerate(cases):
        packed, kw = _inputs(n, bs, dq, 700 + i)
        data.append((n, bs, packed, kw, _oracle(orc, packed, kw, n, bs, "f16")))
    nf4.nf4_set_early_input_reads(True)
    try:
        s = torch.cuda.Stream()
        outs = [torch.empty(max(n for n, *_ in data), dtype=torch.float16, device="cuda") for _ in range(2)]
        dev_in = []
        for n, bs, packed, kw, _ in data:
            dev_in.append((dev(packed), {k: (dev(v) if isinstance(v, np.ndarray) else v) for k, v in kw.items()}))
        torch.cuda.synchronize()
        results = []
        with torch.cuda.stream(s):
            for rep in range(3):
                for i, (n, bs, packed, kw, ref) in enumerate(data):
                    out = outs[(rep * len(data) + i) % 2]
                    out.fill_(0.0)                       # a kernel writing `out` right before the launch
                    pk, k2 = dev_in[i]
                    if dq:
                        d = nf4.DQ(k2["qabsmax"], k2["code2"], k2["absmax2"], k2["offset"])
                        nf4.nf4_dequantize(pk, None, d, n=n, blocksize=bs, out_dtype="f16", out=out[:n], stream=s)
                    else:
                        nf4.nf4_dequantize(pk, k2["absmax"], None, n=n, blocksize=bs, out_dtype="f16", out=out[:n],
                                           stream=s)
                    got = torch.empty(n, dtype=torch.int16, device="cuda")
                    got.copy_(out[:n].view(torch.int16))
                    results.append((rep, i, got, ref))
        s.synchronize()
        for rep, i, got, ref in results:
            assert np.array_equal(got.cpu().numpy().view(np.uint16), ref), (rep, i)
    finally:
        nf4.nf4_set_early_input_reads(False)
