"""Every-element parity at BASELINE.json's full sizes (SURVEY 8(c) item 20:
"compare every 16-bit output word, all elements of all 5 configs").

The paper's correctness claim is bit-exact output for all models (§V-A;
"token-exact compatibility", §IV-A); north_star makes it "bit-exact vs the
CPU oracle on all five configs" at 0 ULP.  Here the CUDA path runs in the launch
configuration bench.py times (WeightStore.dequantize_all: <=128 tensors per
launch; the config-5 sweep: one nf4_dequantize per size), its inputs filled on
the device by the counter-based generator; the oracle gets the SAME inputs
regenerated on the host by synth/hashgen.c (input generation only, pinned to
synth/inputs.py in tests/test_synth_host.py) -- nothing the oracle sees comes
from the CUDA path.  Outputs are copied back in 128 Mi-element chunks and
compared word for word; the element and mismatch counts are logged (one JSON
line per config to $NF4_PARITY_LOG, or stdout).

Inputs are the counter-hash family, not bench.py's default
Gaussian family: the kernel's control flow and launch configuration do not
depend on the values, and only the hash family can be regenerated on the host
at 10^11 elements.
"""
from __future__ import annotations

import json
import os
import time

import numpy as np
import pytest

from synth import fast
from synth import inputs as syn
from synth import workloads as wl

pytestmark = pytest.mark.gpu

CHUNK = 1 << 27          # elements; a multiple of 4096 * 256, so every chunk starts a block group
THREADS = len(os.sched_getaffinity(0))


@pytest.fixture(scope="module")
def nf4():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_02556_b200 as m
    m.load()
    m.nf4_set_max_ctas(0)
    return m


@pytest.fixture(scope="module")
def pinned():
    import torch
    return torch.empty(CHUNK, dtype=torch.int16).pin_memory()


def _log(rec):
    line = json.dumps(rec)
    path = os.environ.get("NF4_PARITY_LOG")
    if path:
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "a") as f:
            f.write(line + "\n")
    print(line)


def _host_inputs(seed, k0, m, bs, dq, code2):
    """Inputs of elements [k0, k0 + m) of the tensor with this seed, as a
    self-contained tensor (k0 is a multiple of bs * 256)."""
    nbc = -(-m // bs)
    b0 = k0 // bs
    packed = fast.packed(seed, k0 // 2, (m + 1) // 2, THREADS)
    if dq:
        return packed, dict(qabsmax=fast.qabsmax(seed, b0, nbc, THREADS), code2=code2,
                            absmax2=fast.absmax2(seed, b0 // 256, -(-nbc // 256), THREADS),
                            offset=float(syn.hash_offset(seed)))
    return packed, dict(absmax=fast.absmax(seed, b0, nbc, THREADS))


def _compare_words(dev_words, ref, pinned):
    """Copy device int16 words to the pinned staging buffer and count mismatches."""
    import torch
    m = dev_words.numel()
    buf = pinned[:m]
    buf.copy_(dev_words)
    torch.cuda.synchronize()
    got = buf.numpy().view(np.uint16)
    return int(np.count_nonzero(got != ref))


def _check_store_full(ws, orc, pinned):
    """Every element of every tensor of the store vs the oracle; returns (elements, mismatches, first)."""
    code = orc.OUT_F16 if ws.out_dtype == "f16" else orc.OUT_BF16
    code2 = syn.dynamic_map_code2()
    elems = bad = 0
    first = None
    for i, e in enumerate(ws.entries):
        for k0 in range(0, e.n, CHUNK):
            m = min(CHUNK, e.n - k0)
            packed, kw = _host_inputs(e.seed, k0, m, ws.blocksize, ws.dq, code2)
            ref = orc.dequantize(packed, m, ws.blocksize, code, threads=THREADS, **kw)
            nb = _compare_words(ws.out_words(i, k0, k0 + m), ref, pinned)
            elems += m
            if nb and first is None:
                first = (e.name, k0)
            bad += nb
    return elems, bad, first


def _run_store(nf4, orc, pinned, key, tensors, seed0, label):
    import torch
    from synth import stores
    c = wl.CONFIGS[key]
    t0 = time.perf_counter()
    ws = stores.from_hash(tensors, c.blocksize, c.dq, c.out_dtype, seed0=seed0, device="cuda")
    ws.out.fill_(0x7F)                       # no stale output can pass
    launches = ws.dequantize_all()
    torch.cuda.synchronize()
    elems, bad, first = _check_store_full(ws, orc, pinned)
    rec = {"test": "full_parity", "config": key, "what": label, "tensors": len(tensors), "launches": launches,
           "elements_compared": elems, "elements_expected": ws.n_total, "mismatches": bad, "first_mismatch": first,
           "oracle_threads": THREADS, "seconds": round(time.perf_counter() - t0, 1)}
    _log(rec)
    del ws
    torch.cuda.empty_cache()
    assert elems == rec["elements_expected"]
    assert bad == 0, rec


@pytest.mark.parametrize("key", ["cfg1", "cfg2", "cfg3"])
def test_every_element_single_gpu_configs(nf4, orc, pinned, key):
    """Configs 1-3 in full: one 4096x4096 tensor; Gemma-3-27B's 434 weights
    (25.6 G elements); Qwen3-32B's 448 weights (31.2 G elements)."""
    _run_store(nf4, orc, pinned, key, wl.config_tensors(key), 1000 * int(key[-1]), "all tensors")


def test_every_element_llama_all_eight_row_shards(nf4, orc, pinned):
    """Config 4: Llama-3.3-70B row-sharded 8 ways; each rank's shard set
    (8.56 G elements, bench.py's seeds for that rank) runs in turn on this GPU."""
    for rank in range(8):
        _run_store(nf4, orc, pinned, "cfg4", wl.config_tensors("cfg4", world_size=8, rank=rank),
                   4000 + 100000 * rank, f"rank {rank} of 8")


@pytest.mark.parametrize("dq", [False, True])
@pytest.mark.parametrize("bs", [64, 128, 256, 4096])
def test_every_element_config5_sweep(nf4, orc, pinned, bs, dq):
    """Config 5: n = 2^20 .. 2^30 (11 sizes) x fp16/bf16 at this blocksize and
    absmax mode, one nf4_dequantize per size (the sweep's launch).  The tensor of
    size n is the first n elements of one 2^30-element counter-hash tensor, so
    one oracle pass over 2^30 elements is the reference for every size."""
    import torch
    from paper_2604_02556_b200 import _lib
    N = 1 << 30
    seed = 5000 + 10 * bs + int(dq)
    nb = N // bs
    packed = torch.empty(N // 2, dtype=torch.uint8, device="cuda")
    nf4.nf4_synth_fill(_lib.NF4_SYNTH_CODES, seed, 0, N // 2, packed)
    if dq:
        q = torch.empty(nb, dtype=torch.uint8, device="cuda")
        a2 = torch.empty(-(-nb // 256), dtype=torch.float32, device="cuda")
        nf4.nf4_synth_fill(_lib.NF4_SYNTH_QABSMAX, seed, 0, nb, q)
        nf4.nf4_synth_fill(_lib.NF4_SYNTH_ABSMAX2, seed, 0, a2.numel(), a2)
        code2 = syn.dynamic_map_code2()
        dqs = nf4.DQ(q, torch.from_numpy(code2).cuda(), a2, float(syn.hash_offset(seed)))
        absmax = None
    else:
        absmax = torch.empty(nb, dtype=torch.float32, device="cuda")
        nf4.nf4_synth_fill(_lib.NF4_SYNTH_ABSMAX, seed, 0, nb, absmax)
        dqs, code2 = None, None
    out = torch.empty(N, dtype=torch.int16, device="cuda")
    sizes = [1 << p for p in range(20, 31)]
    for dtype in ("f16", "bf16"):
        code = orc.OUT_F16 if dtype == "f16" else orc.OUT_BF16
        t0 = time.perf_counter()
        refs = []
        for k0 in range(0, N, CHUNK):
            pk, kw = _host_inputs(seed, k0, CHUNK, bs, dq, code2)
            refs.append(orc.dequantize(pk, CHUNK, bs, code, threads=THREADS, **kw))
        elems = bad = 0
        per_size = {}
        for n in sizes:
            out.fill_(0x7F7F)
            nf4.nf4_dequantize(packed, absmax, dqs, n=n, blocksize=bs, out_dtype=dtype,
                               out=out.view(torch.float16 if dtype == "f16" else torch.bfloat16))
            nbad = 0
            for ci, k0 in enumerate(range(0, n, CHUNK)):
                m = min(CHUNK, n - k0)
                nbad += _compare_words(out[k0:k0 + m], refs[ci][:m], pinned)
            # nothing written past out[n - 1]
            if n < N:
                tail = out[n:n + 4096].cpu().numpy()
                nbad += int(np.count_nonzero(tail != 0x7F7F))
            per_size[n] = nbad
            elems += n
            bad += nbad
        _log({"test": "full_parity", "config": "cfg5", "blocksize": bs, "absmax": "double-quant" if dq else "fp32",
              "out_dtype": dtype, "sizes": f"2^20..2^30 ({len(sizes)})", "elements_compared": elems,
              "mismatches": bad, "oracle_threads": THREADS, "seconds": round(time.perf_counter() - t0, 1)})
        assert bad == 0, {k: v for k, v in per_size.items() if v}
    del packed, out
    torch.cuda.empty_cache()


def test_row_shards_equal_slices_of_flat_result(nf4, orc, pinned):
    """SURVEY §4 T10 (multi-GPU without a cluster): a globally quantized weight
    dequantized flat, and its G row shards dequantized one by one from slices of
    the same codes / scales (shard boundaries are multiples of 16384 = 64 * 256
    elements, so they align with both quantization levels), give identical
    bytes -- what G GPUs would produce, byte for byte.  Llama gate_proj
    [28672 x 8192] (235 M elements), G = 2, 4, 8, double-quant and fp32 absmax."""
    import torch
    from paper_2604_02556_b200 import _lib
    rows, cols = 28672, 8192
    n = rows * cols
    bs = 64
    nb = n // bs
    seed = 4242
    packed = torch.empty(n // 2, dtype=torch.uint8, device="cuda")
    nf4.nf4_synth_fill(_lib.NF4_SYNTH_CODES, seed, 0, n // 2, packed)
    q = torch.empty(nb, dtype=torch.uint8, device="cuda")
    a2 = torch.empty(nb // 256, dtype=torch.float32, device="cuda")
    absmax = torch.empty(nb, dtype=torch.float32, device="cuda")
    nf4.nf4_synth_fill(_lib.NF4_SYNTH_QABSMAX, seed, 0, nb, q)
    nf4.nf4_synth_fill(_lib.NF4_SYNTH_ABSMAX2, seed, 0, nb // 256, a2)
    nf4.nf4_synth_fill(_lib.NF4_SYNTH_ABSMAX, seed, 0, nb, absmax)
    code2 = torch.from_numpy(syn.dynamic_map_code2()).cuda()
    off = float(syn.hash_offset(seed))
    for dq in (True, False):
        flat = nf4.nf4_dequantize(packed, None if dq else absmax, nf4.DQ(q, code2, a2, off) if dq else None,
                                  n=n, blocksize=bs, out_dtype="bf16")
        for G in (2, 4, 8):
            sh = n // G
            assert sh % 16384 == 0
            shards = torch.full((n,), 0x7F7F, dtype=torch.int16, device="cuda")
            for r in range(G):
                k0 = r * sh
                dqs = nf4.DQ(q[k0 // bs:(k0 + sh) // bs], code2, a2[k0 // bs // 256:(k0 + sh) // bs // 256], off) \
                    if dq else None
                nf4.nf4_dequantize(packed[k0 // 2:(k0 + sh) // 2], None if dq else absmax[k0 // bs:(k0 + sh) // bs],
                                   dqs, n=sh, blocksize=bs, out_dtype="bf16",
                                   out=shards[k0:k0 + sh].view(torch.bfloat16))
            torch.cuda.synchronize()
            assert torch.equal(shards, flat.view(torch.int16)), (dq, G)
        # and the flat result is the oracle's (sampled 1 M elements at 3 offsets)
        code2h = syn.dynamic_map_code2()
        for k0 in (0, n // 2 + (1 << 20), n - (1 << 20)):
            pk, kw = _host_inputs(seed, k0, 1 << 20, bs, dq, code2h)
            ref = orc.dequantize(pk, 1 << 20, bs, orc.OUT_BF16, threads=THREADS, **kw)
            assert _compare_words(flat.view(torch.int16)[k0:k0 + (1 << 20)], ref, pinned) == 0
    del packed, q, a2, absmax
    torch.cuda.empty_cache()
