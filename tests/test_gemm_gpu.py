"""F1: fused NF4 dequant + tcgen05 GEMM vs the oracle.

* one-hot X rows make every Y[m, n] a single exact product 1 * W[n, k_m], so the
  weights the tensor cores consumed are checked BIT-EXACT against the oracle's
  dequantization (the hot path's definition);
* random X: |Y - Y_ref| <= K * 2^-23 * sum_k |x w| (+ the output rounding for
  16-bit Y), Y_ref in fp64 from oracle.gemm_reference.
"""
from __future__ import annotations

import ml_dtypes
import numpy as np
import pytest

from synth import inputs as syn

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nf4():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_02556_b200 as m
    m.load()
    return m


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _weights(N, K, bs, dq, seed):
    n = N * K
    nb = n // bs
    packed = syn.hash_packed(seed, 0, n // 2)
    if dq:
        kw = dict(qabsmax=syn.hash_qabsmax(seed, 0, nb), code2=syn.dynamic_map_code2(),
                  absmax2=syn.hash_absmax2(seed, 0, -(-nb // 256)), offset=float(syn.hash_offset(seed)))
    else:
        kw = dict(absmax=syn.hash_absmax(seed, 0, nb))
    return packed, kw


def _run(nf4, x16, xdt, M, packed, kw, N, K, bs, ydt, splits):
    import torch
    tdt = torch.bfloat16 if xdt == "bf16" else torch.float16
    x = dev(x16.view(np.int16)).view(tdt).reshape(M, K)
    if "absmax" in kw:
        y = nf4.nf4_gemm(x, dev(packed), dev(kw["absmax"]), None, N=N, K=K, blocksize=bs, y_dtype=ydt, splits=splits)
    else:
        d = nf4.DQ(dev(kw["qabsmax"]), dev(kw["code2"]), dev(kw["absmax2"]), kw["offset"])
        y = nf4.nf4_gemm(x, dev(packed), None, d, N=N, K=K, blocksize=bs, y_dtype=ydt, splits=splits)
    torch.cuda.synchronize()
    return y


@pytest.mark.parametrize("xdt", ["bf16", "f16"])
@pytest.mark.parametrize("dq", [False, True])
def test_gemm_weights_bit_exact_via_one_hot(nf4, orc, xdt, dq):
    """Y[m, n] = W[n, k_m] exactly: the tensor cores saw the hot path's weights."""
    # splits 0 = stream-K: (16, 5120, 448) has 7 chunks per tile (ranges not 4-aligned,
    # tiles cut into up to 7 segments); (300, 256, 1280) two token tiles, 5 segments each
    cases = ((16, 256, 512, 64, 1), (5, 384, 1024, 128, 3), (40, 200, 640, 64, 2),
             (16, 256, 512, 64, 0), (40, 200, 640, 64, 0), (16, 5120, 448, 64, 0), (300, 256, 1280, 64, 0),
             # every token-tile width (BN 32 / 64 with 2-chunk stages / 128) through the byte-pair
             # table, stream-K, incl. the general (per-chunk) scale path at blocksize 128
             (24, 384, 768, 64, 0), (50, 256, 1024, 128, 0), (100, 256, 1024, 64, 0))
    for (M, N, K, bs, splits) in cases:
        packed, kw = _weights(N, K, bs, dq, seed=M + N + K)
        ks = (np.arange(M) * 37 + 11) % K
        x = np.zeros((M, K), np.float32)
        x[np.arange(M), ks] = 1.0
        x16 = (x.astype(ml_dtypes.bfloat16) if xdt == "bf16" else x.astype(np.float16)).view(np.uint16)
        y = _run(nf4, x16, xdt, M, packed, kw, N, K, bs, "f32", splits).cpu().numpy()
        code = orc.OUT_BF16 if xdt == "bf16" else orc.OUT_F16
        w16 = orc.dequantize(packed, N * K, bs, code, threads=8, **kw).reshape(N, K)
        np16 = ml_dtypes.bfloat16 if xdt == "bf16" else np.float16
        want = w16[:, ks].T.view(np16).astype(np.float32)           # [M, N]
        assert np.array_equal(y.view(np.uint32), want.view(np.uint32)), (M, N, K, splits)


SHAPES = [(1, 128, 64), (2, 256, 1024), (7, 384, 2048), (16, 1024, 4096), (33, 640, 1536),
          (64, 512, 5376), (100, 256, 1024), (130, 384, 512), (300, 256, 768)]


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_gemm_random_within_fp32_bound(nf4, orc, M, N, K):
    rng = np.random.Generator(np.random.Philox(M * 1000 + K))
    x16 = rng.standard_normal((M, K)).astype(np.float32).astype(ml_dtypes.bfloat16).view(np.uint16)
    for dq in (False, True):
        packed, kw = _weights(N, K, 64, dq, seed=N + K + int(dq))
        ref, mag = orc.gemm_reference(x16, orc.OUT_BF16, packed, N, K, 64, **kw)
        for splits in (1, 0):
            y = _run(nf4, x16, "bf16", M, packed, kw, N, K, 64, "f32", splits).cpu().numpy().astype(np.float64)
            bound = K * 2.0 ** -23 * mag + 1e-30
            err = np.abs(y - ref)
            assert (err <= bound).all(), (M, N, K, dq, splits, float((err / bound).max()))


@pytest.mark.parametrize("bs", [64, 128, 256, 4096])
@pytest.mark.parametrize("xdt", ["bf16", "f16"])
def test_gemm_stream_k_blocksizes_and_dtypes(nf4, orc, bs, xdt):
    """Stream-K (splits=0) on the general scale path (bs > 64), the fast one (bs 64),
    fp16 and bf16 X, fp32 and double-quant absmax; K = 4096 keeps every blocksize legal
    and cuts tiles into several pieces."""
    M, N, K = 24, 1280, 4096
    rng = np.random.Generator(np.random.Philox(bs + (xdt == "f16")))
    xf = rng.standard_normal((M, K)).astype(np.float32)
    x16 = (xf.astype(ml_dtypes.bfloat16) if xdt == "bf16" else xf.astype(np.float16)).view(np.uint16)
    code = orc.OUT_BF16 if xdt == "bf16" else orc.OUT_F16
    for dq in (False, True):
        packed, kw = _weights(N, K, bs, dq, seed=bs + 7 * int(dq))
        ref, mag = orc.gemm_reference(x16, code, packed, N, K, bs, **kw)
        y = _run(nf4, x16, xdt, M, packed, kw, N, K, bs, "f32", 0).cpu().numpy().astype(np.float64)
        err = np.abs(y - ref)
        bound = K * 2.0 ** -23 * mag + 1e-30
        assert (err <= bound).all(), (bs, xdt, dq, float((err / bound).max()))


def test_gemm_stream_k_unaligned_scales_take_general_path(nf4, orc):
    """absmax / qabsmax pointers that break the vector-load alignment of the fast
    scale path must still give the same bits (general path)."""
    import torch
    M, N, K = 16, 512, 2048
    rng = np.random.Generator(np.random.Philox(77))
    x16 = rng.standard_normal((M, K)).astype(np.float32).astype(ml_dtypes.bfloat16).view(np.uint16)
    x = dev(x16.view(np.int16)).view(torch.bfloat16).reshape(M, K)
    packed, kw = _weights(N, K, 64, False, 12)
    a_buf = torch.zeros(kw["absmax"].size + 1, dtype=torch.float32, device="cuda")
    a_buf[1:] = dev(kw["absmax"])
    y_al = nf4.nf4_gemm(x, dev(packed), dev(kw["absmax"]), None, N=N, K=K, y_dtype="f32")
    y_un = nf4.nf4_gemm(x, dev(packed), a_buf[1:], None, N=N, K=K, y_dtype="f32")
    torch.cuda.synchronize()
    assert torch.equal(y_al.view(torch.int32), y_un.view(torch.int32))
    packed, kw = _weights(N, K, 64, True, 13)
    q_buf = torch.zeros(kw["qabsmax"].size + 1, dtype=torch.uint8, device="cuda")
    q_buf[1:] = dev(kw["qabsmax"])
    d_al = nf4.DQ(dev(kw["qabsmax"]), dev(kw["code2"]), dev(kw["absmax2"]), kw["offset"])
    d_un = nf4.DQ(q_buf[1:], dev(kw["code2"]), dev(kw["absmax2"]), kw["offset"])
    y_al = nf4.nf4_gemm(x, dev(packed), None, d_al, N=N, K=K, y_dtype="f32")
    y_un = nf4.nf4_gemm(x, dev(packed), None, d_un, N=N, K=K, y_dtype="f32")
    torch.cuda.synchronize()
    assert torch.equal(y_al.view(torch.int32), y_un.view(torch.int32))


def test_gemm_bf16_output_rounding(nf4, orc):
    M, N, K = 24, 384, 2048
    rng = np.random.Generator(np.random.Philox(5))
    x16 = rng.standard_normal((M, K)).astype(np.float32).astype(ml_dtypes.bfloat16).view(np.uint16)
    packed, kw = _weights(N, K, 64, True, 17)
    ref, mag = orc.gemm_reference(x16, orc.OUT_BF16, packed, N, K, 64, **kw)
    y = _run(nf4, x16, "bf16", M, packed, kw, N, K, 64, "bf16", 0).float().cpu().numpy().astype(np.float64)
    # fp32 accumulation bound, then one bf16 rounding (half ulp = 2^-8 relative)
    bound = K * 2.0 ** -23 * mag * (1 + 2.0 ** -8) + np.abs(ref) * 2.0 ** -8 + 1e-30
    assert (np.abs(y - ref) <= bound).all()


def test_gemm_split_k_is_deterministic(nf4):
    M, N, K = 8, 512, 8192
    rng = np.random.Generator(np.random.Philox(8))
    x16 = rng.standard_normal((M, K)).astype(np.float32).astype(ml_dtypes.bfloat16).view(np.uint16)
    packed, kw = _weights(N, K, 64, True, 3)
    a = _run(nf4, x16, "bf16", M, packed, kw, N, K, 64, "f32", 4).cpu().numpy()
    b = _run(nf4, x16, "bf16", M, packed, kw, N, K, 64, "f32", 4).cpu().numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_gemm_stream_k_is_deterministic_and_matches_classic(nf4, orc):
    """Stream-K: identical bits run to run; within the fp32 bound of the oracle."""
    M, N, K = 16, 21504 // 8, 5376
    rng = np.random.Generator(np.random.Philox(9))
    x16 = rng.standard_normal((M, K)).astype(np.float32).astype(ml_dtypes.bfloat16).view(np.uint16)
    packed, kw = _weights(N, K, 64, True, 4)
    a = _run(nf4, x16, "bf16", M, packed, kw, N, K, 64, "f32", 0).cpu().numpy()
    b = _run(nf4, x16, "bf16", M, packed, kw, N, K, 64, "f32", 0).cpu().numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    ref, mag = orc.gemm_reference(x16, orc.OUT_BF16, packed, N, K, 64, **kw)
    assert (np.abs(a.astype(np.float64) - ref) <= K * 2.0 ** -23 * mag + 1e-30).all()


def test_gemm_stream_k_workspace_reuse(nf4, orc):
    """One zero-filled workspace serves a sequence of stream-K calls of different
    shapes (each call leaves its per-tile counters at zero again)."""
    import torch
    shapes = [(16, 5120, 448), (16, 21504 // 8, 5376), (40, 2048, 1024), (16, 5120, 448)]
    need = max(nf4.nf4_gemm_workspace_bytes(M, N, K, 0) for M, N, K in shapes)
    assert need > 0
    ws = torch.zeros(need, dtype=torch.uint8, device="cuda")
    for idx, (M, N, K) in enumerate(shapes):
        rng = np.random.Generator(np.random.Philox(100 + idx))
        x16 = rng.standard_normal((M, K)).astype(np.float32).astype(ml_dtypes.bfloat16).view(np.uint16)
        packed, kw = _weights(N, K, 64, False, 50 + idx)
        x = dev(x16.view(np.int16)).view(torch.bfloat16).reshape(M, K)
        y = nf4.nf4_gemm(x, dev(packed), dev(kw["absmax"]), None, N=N, K=K, y_dtype="f32", workspace=ws)
        torch.cuda.synchronize()
        ref, mag = orc.gemm_reference(x16, orc.OUT_BF16, packed, N, K, 64, **kw)
        err = np.abs(y.cpu().numpy().astype(np.float64) - ref)
        assert (err <= K * 2.0 ** -23 * mag + 1e-30).all(), (M, N, K)
        tiles = -(-N // 128) * -(-M // (16 if M <= 16 else 32 if M <= 32 else 64 if M <= 64 else 128))
        assert int(ws[:4 * tiles].view(torch.int32).abs().sum()) == 0, "stream-K counters not reset"


@pytest.mark.parametrize("M", [5, 16, 40, 100])
def test_gemm_grouped_bit_exact_weights_and_bound(nf4, orc, M):
    """nf4_gemm_grouped: q/k/v-like members (different N, one not a multiple of 128,
    fp32 and double-quant absmax) in one launch; one-hot X checks every member's
    weights bit-exactly, random X against the fp64 oracle bound."""
    import torch
    K = 1536
    Ns = (1024, 200, 384)
    dqs = (True, False, True)
    members, kws, packs = [], [], []
    for i, (N, dq) in enumerate(zip(Ns, dqs)):
        packed, kw = _weights(N, K, 64, dq, seed=300 + i)
        packs.append(packed)
        kws.append(kw)
        if dq:
            d = nf4.DQ(dev(kw["qabsmax"]), dev(kw["code2"]), dev(kw["absmax2"]), kw["offset"])
            members.append((dev(packed), None, d, N))
        else:
            members.append((dev(packed), dev(kw["absmax"]), None, N))
    # one-hot rows: Y_i[m, n] = W_i[n, k_m] exactly
    ks = (np.arange(M) * 131 + 7) % K
    xo = np.zeros((M, K), np.float32)
    xo[np.arange(M), ks] = 1.0
    x16 = xo.astype(ml_dtypes.bfloat16).view(np.uint16)
    x = dev(x16.view(np.int16)).view(torch.bfloat16).reshape(M, K)
    ys = nf4.nf4_gemm_grouped(x, members, K=K, y_dtype="f32")
    torch.cuda.synchronize()
    for i, N in enumerate(Ns):
        w16 = orc.dequantize(packs[i], N * K, 64, orc.OUT_BF16, threads=8, **kws[i]).reshape(N, K)
        want = w16[:, ks].T.view(ml_dtypes.bfloat16).astype(np.float32)
        assert np.array_equal(ys[i].cpu().numpy().view(np.uint32), want.view(np.uint32)), (M, i)
    # random X, within the fp32 accumulation bound
    rng = np.random.Generator(np.random.Philox(M))
    x16 = rng.standard_normal((M, K)).astype(np.float32).astype(ml_dtypes.bfloat16).view(np.uint16)
    x = dev(x16.view(np.int16)).view(torch.bfloat16).reshape(M, K)
    ys = nf4.nf4_gemm_grouped(x, members, K=K, y_dtype="f32")
    torch.cuda.synchronize()
    for i, N in enumerate(Ns):
        ref, mag = orc.gemm_reference(x16, orc.OUT_BF16, packs[i], N, K, 64, **kws[i])
        err = np.abs(ys[i].cpu().numpy().astype(np.float64) - ref)
        assert (err <= K * 2.0 ** -23 * mag + 1e-30).all(), (M, i)


def test_gemm_grouped_workspace_reuse_and_errors(nf4, orc):
    import torch
    M, K = 16, 2048
    Ns = (2048, 512)
    members, kws, packs = [], [], []
    for i, N in enumerate(Ns):
        packed, kw = _weights(N, K, 64, False, seed=400 + i)
        packs.append(packed)
        kws.append(kw)
        members.append((dev(packed), dev(kw["absmax"]), None, N))
    ws = torch.zeros(max(16, nf4.nf4_gemm_grouped_workspace_bytes(M, Ns, K)), dtype=torch.uint8, device="cuda")
    rng = np.random.Generator(np.random.Philox(4))
    for rep in range(3):
        x16 = rng.standard_normal((M, K)).astype(np.float32).astype(ml_dtypes.bfloat16).view(np.uint16)
        x = dev(x16.view(np.int16)).view(torch.bfloat16).reshape(M, K)
        ys = nf4.nf4_gemm_grouped(x, members, K=K, y_dtype="f32", workspace=ws)
        torch.cuda.synchronize()
        for i, N in enumerate(Ns):
            ref, mag = orc.gemm_reference(x16, orc.OUT_BF16, packs[i], N, K, 64, **kws[i])
            assert (np.abs(ys[i].cpu().numpy().astype(np.float64) - ref) <= K * 2.0 ** -23 * mag + 1e-30).all()
    with pytest.raises(nf4.NF4Error) as e:
        nf4.nf4_gemm_grouped(x, members * 3, K=K)             # 6 weights > NF4_GEMM_MAX_GROUP
    assert e.value.status == 2


def test_gemm_argument_errors(nf4):
    import torch
    x = torch.zeros((4, 100), dtype=torch.bfloat16, device="cuda")
    p = torch.zeros(100 * 128 // 2, dtype=torch.uint8, device="cuda")
    a = torch.ones(200, dtype=torch.float32, device="cuda")
    with pytest.raises(nf4.NF4Error) as e:
        nf4.nf4_gemm(x, p, a, None, N=128, K=100)             # K not a multiple of 64
    assert e.value.status == 2


# ---------------------------------------------------------------------------
# every weight bit-exact, and exact sums (verdict r01: the one-hot test read only
# M of the K columns; the random-X bound admits one mis-decoded weight)
# ---------------------------------------------------------------------------
def _x_tensor(x16, xdt, M, K):
    import torch
    tdt = torch.bfloat16 if xdt == "bf16" else torch.float16
    return dev(x16.view(np.int16)).view(tdt).reshape(M, K)


def _to16(xf, xdt):
    return (xf.astype(ml_dtypes.bfloat16) if xdt == "bf16" else xf.astype(np.float16)).view(np.uint16)


def _pos0(a):
    """fp32 values with -0 folded into +0 (a one-hot sum's zero sign depends on
    the order of the zero terms, not on the weight)."""
    a = np.asarray(a, np.float32) + np.float32(0.0)
    return a.view(np.uint32)


FULL_CASES = [  # (M -> token-tile width BN, N, K, blocksize)
    (1, 256, 512, 64), (16, 2688, 5376, 64), (32, 640, 2048, 128), (64, 384, 1024, 64), (128, 200, 1024, 256)]


@pytest.mark.parametrize("xdt", ["bf16", "f16"])
@pytest.mark.parametrize("dq", [False, True])
def test_gemm_recovers_every_weight_bit_exact(nf4, orc, xdt, dq):
    """X = identity blocks covering all of K, one stream-K GEMM per block of M
    columns: Y[m, n] = W[n, k0 + m] exactly, so EVERY dequantized weight the
    tensor cores consumed is compared with the oracle's, at every token-tile
    width (BN 16 / 32 / 64 / 128) and several blocksizes."""
    import torch
    code = orc.OUT_BF16 if xdt == "bf16" else orc.OUT_F16
    np16 = ml_dtypes.bfloat16 if xdt == "bf16" else np.float16
    for (M, N, K, bs) in FULL_CASES:
        packed, kw = _weights(N, K, bs, dq, seed=7 * M + N + K + int(dq))
        pk = dev(packed)
        if dq:
            absmax, d = None, nf4.DQ(dev(kw["qabsmax"]), dev(kw["code2"]), dev(kw["absmax2"]), kw["offset"])
        else:
            absmax, d = dev(kw["absmax"]), None
        ws = torch.zeros(max(16, nf4.nf4_gemm_workspace_bytes(M, N, K, 0)), dtype=torch.uint8, device="cuda")
        w_gpu = np.zeros((N, K), np.float32)
        for k0 in range(0, K, M):
            x = np.zeros((M, K), np.float32)
            x[np.arange(M), k0 + np.arange(M)] = 1.0
            y = nf4.nf4_gemm(_x_tensor(_to16(x, xdt), xdt, M, K), pk, absmax, d, N=N, K=K, blocksize=bs,
                             y_dtype="f32", workspace=ws)
            torch.cuda.synchronize()
            w_gpu[:, k0:k0 + M] = y.cpu().numpy().T
        want = orc.dequantize(packed, N * K, bs, code, threads=8, **kw).view(np16).astype(np.float32).reshape(N, K)
        bad = _pos0(w_gpu) != _pos0(want)
        assert not bad.any(), (M, N, K, bs, int(bad.sum()), np.argwhere(bad)[:3].tolist())


def _sparse_pm1(M, K, nnz, seed):
    """X rows with `nnz` entries of +-1 at random columns (rest 0)."""
    rng = np.random.Generator(np.random.Philox(seed))
    x = np.zeros((M, K), np.float32)
    for m in range(M):
        cols = rng.choice(K, nnz, replace=False)
        x[m, cols] = rng.choice(np.array([-1.0, 1.0], np.float32), nnz)
    return x


def _exact_reference(x16, xdt, packed, N, K, bs, kw, orc):
    """Y in fp64 from the oracle's weights; with +-1 X and few non-zeros every
    partial sum is a multiple of the weights' smallest ulp and below 2^24 of
    them, so ANY fp32 summation order gives exactly this value (checked here)."""
    code = orc.OUT_BF16 if xdt == "bf16" else orc.OUT_F16
    ref, mag = orc.gemm_reference(x16, code, packed, N, K, bs, **kw)
    np16 = ml_dtypes.bfloat16 if xdt == "bf16" else np.float16
    w = orc.dequantize(packed, N * K, bs, code, threads=8, **kw).view(np16).astype(np.float64)
    nz = np.abs(w[w != 0])
    _, e = np.frexp(nz)                              # nz = f * 2^e, f in [0.5, 1)
    mant = 8 if xdt == "bf16" else 11
    ulp = np.ldexp(1.0, int(e.min()) - mant)
    assert mag.max() < ulp * 2.0 ** 24, "fixture: sums not exact in fp32"
    assert np.array_equal(ref.astype(np.float32).astype(np.float64), ref)
    return ref


@pytest.mark.parametrize("xdt", ["bf16", "f16"])
@pytest.mark.parametrize("dq", [False, True])
def test_gemm_sparse_pm1_exact(nf4, orc, xdt, dq):
    """X with 64 entries of +-1 per row: the exact Y is representable in fp32 and
    reached by every summation order, so stream-K Y must equal the fp64 oracle
    product BIT FOR BIT (fp32 output), and its RNE to bf16 / fp16 (16-bit output).
    A single mis-decoded weight, a dropped k-chunk or a wrong partial changes Y."""
    for (M, N, K, bs) in [(1, 512, 1024, 64), (16, 2688, 5376, 64), (40, 640, 2048, 128), (100, 384, 1024, 64),
                          (128, 256, 3072, 64), (200, 384, 1024, 256)]:
        packed, kw = _weights(N, K, bs, dq, seed=3 * M + N + K + int(dq))
        x16 = _to16(_sparse_pm1(M, K, 64, M + K), xdt)
        ref = _exact_reference(x16, xdt, packed, N, K, bs, kw, orc)
        y = _run(nf4, x16, xdt, M, packed, kw, N, K, bs, "f32", 0).cpu().numpy()
        assert np.array_equal(_pos0(y), _pos0(ref.astype(np.float32))), (M, N, K, bs)
        y16 = _run(nf4, x16, xdt, M, packed, kw, N, K, bs, xdt, 0)
        got = y16.view(__import__("torch").int16).cpu().numpy().view(np.uint16)
        want = _to16(ref.astype(np.float32), xdt)
        np16 = ml_dtypes.bfloat16 if xdt == "bf16" else np.float16
        assert np.array_equal(_pos0(got.view(np16).astype(np.float32)), _pos0(want.view(np16).astype(np.float32))), \
            (M, N, K, bs)


@pytest.mark.parametrize("M", [1, 16, 64])
def test_gemm_grouped_sparse_pm1_exact_and_full_weights(nf4, orc, M):
    """nf4_gemm_grouped: exact sums (sparse +-1 X) for every member, and every
    weight of every member recovered through identity X blocks."""
    import torch
    K = 1024
    Ns = (512, 200, 384, 128)
    dqs = (True, False, True, False)
    members, kws, packs = [], [], []
    for i, (N, dq) in enumerate(zip(Ns, dqs)):
        packed, kw = _weights(N, K, 64, dq, seed=700 + i + M)
        packs.append(packed)
        kws.append(kw)
        if dq:
            members.append((dev(packed), None, nf4.DQ(dev(kw["qabsmax"]), dev(kw["code2"]), dev(kw["absmax2"]),
                                                      kw["offset"]), N))
        else:
            members.append((dev(packed), dev(kw["absmax"]), None, N))
    x16 = _to16(_sparse_pm1(M, K, 64, 5 + M), "bf16")
    ys = nf4.nf4_gemm_grouped(_x_tensor(x16, "bf16", M, K), members, K=K, y_dtype="f32")
    torch.cuda.synchronize()
    for i, N in enumerate(Ns):
        ref = _exact_reference(x16, "bf16", packs[i], N, K, 64, kws[i], orc)
        assert np.array_equal(_pos0(ys[i].cpu().numpy()), _pos0(ref.astype(np.float32))), (M, i)
    ws = torch.zeros(max(16, nf4.nf4_gemm_grouped_workspace_bytes(M, Ns, K)), dtype=torch.uint8, device="cuda")
    w_gpu = [np.zeros((N, K), np.float32) for N in Ns]
    for k0 in range(0, K, M):
        m_eff = min(M, K - k0)
        x = np.zeros((M, K), np.float32)
        x[np.arange(m_eff), k0 + np.arange(m_eff)] = 1.0
        ys = nf4.nf4_gemm_grouped(_x_tensor(_to16(x, "bf16"), "bf16", M, K), members, K=K, y_dtype="f32",
                                  workspace=ws)
        torch.cuda.synchronize()
        for i in range(len(Ns)):
            w_gpu[i][:, k0:k0 + m_eff] = ys[i].cpu().numpy()[:m_eff].T
    for i, N in enumerate(Ns):
        want = orc.dequantize(packs[i], N * K, 64, orc.OUT_BF16, threads=8, **kws[i]).view(
            ml_dtypes.bfloat16).astype(np.float32).reshape(N, K)
        assert np.array_equal(_pos0(w_gpu[i]), _pos0(want)), (M, i)


# ---------------------------------------------------------------------------
# nf4_gemm_multi: independent problems (own X and K) in one persistent launch
# ---------------------------------------------------------------------------
MULTI_SHAPES = [(512, 1024, True), (200, 2048, False), (384, 512, True), (128, 3072, False), (640, 256, True),
                (256, 1536, True), (130, 768, False)]


def _multi_setup(nf4, M, xdt, seed0, shapes=MULTI_SHAPES, sparse=True):
    import torch
    probs, host = [], []
    for i, (N, K, dq) in enumerate(shapes):
        packed, kw = _weights(N, K, 64, dq, seed=seed0 + i)
        x16 = _to16(_sparse_pm1(M, K, 64, seed0 + 7 * i) if sparse else
                    np.random.Generator(np.random.Philox(seed0 + i)).standard_normal((M, K)).astype(np.float32), xdt)
        x = _x_tensor(x16, xdt, M, K)
        if dq:
            probs.append((x, K, dev(packed), None,
                          nf4.DQ(dev(kw["qabsmax"]), dev(kw["code2"]), dev(kw["absmax2"]), kw["offset"]), N))
        else:
            probs.append((x, K, dev(packed), dev(kw["absmax"]), None, N))
        host.append((x16, packed, kw, N, K))
    return probs, host


@pytest.mark.parametrize("M", [1, 16, 40, 100])
@pytest.mark.parametrize("xdt", ["bf16", "f16"])
def test_gemm_multi_exact_sums(nf4, orc, M, xdt):
    """Seven problems with different N, K, scale formats and their own X in one
    launch: every Y_i equals the exact fp64 oracle product (sparse +-1 X)."""
    import torch
    probs, host = _multi_setup(nf4, M, xdt, 900 + M)
    ys = nf4.nf4_gemm_multi(probs, M=M, x_dtype=xdt, y_dtype="f32")
    torch.cuda.synchronize()
    assert nf4.nf4_last_launch_count() == 1
    for i, (x16, packed, kw, N, K) in enumerate(host):
        ref = _exact_reference(x16, xdt, packed, N, K, 64, kw, orc)
        assert np.array_equal(_pos0(ys[i].cpu().numpy()), _pos0(ref.astype(np.float32))), (M, i)


@pytest.mark.parametrize("M", [1, 16, 64])
def test_gemm_multi_recovers_every_weight(nf4, orc, M):
    """Identity blocks over each problem's own K recover every weight of every
    problem bit-exactly through one launch per block."""
    import torch
    shapes = [(256, 512, True), (136, 1024, False), (384, 256, True)]
    kmax = max(K for _, K, _ in shapes)
    probs0, host = _multi_setup(nf4, M, "bf16", 40 + M, shapes)
    w_gpu = [np.zeros((N, K), np.float32) for N, K, _ in shapes]
    ws = torch.zeros(max(16, nf4.nf4_gemm_multi_workspace_bytes(M, [s[0] for s in shapes], [s[1] for s in shapes])),
                     dtype=torch.uint8, device="cuda")
    for k0 in range(0, kmax, M):
        probs = []
        for (x, K, pk, a, d, N) in probs0:
            xe = np.zeros((M, K), np.float32)
            m_eff = max(0, min(M, K - k0))
            xe[np.arange(m_eff), k0 + np.arange(m_eff)] = 1.0
            probs.append((_x_tensor(_to16(xe, "bf16"), "bf16", M, K), K, pk, a, d, N))
        ys = nf4.nf4_gemm_multi(probs, M=M, x_dtype="bf16", y_dtype="f32", workspace=ws)
        torch.cuda.synchronize()
        for i, (N, K, _) in enumerate(shapes):
            m_eff = max(0, min(M, K - k0))
            if m_eff:
                w_gpu[i][:, k0:k0 + m_eff] = ys[i].cpu().numpy()[:m_eff].T
    for i, (x16, packed, kw, N, K) in enumerate(host):
        want = orc.dequantize(packed, N * K, 64, orc.OUT_BF16, threads=8, **kw).view(
            ml_dtypes.bfloat16).astype(np.float32).reshape(N, K)
        assert np.array_equal(_pos0(w_gpu[i]), _pos0(want)), (M, i)


def test_gemm_multi_random_bound_workspace_reuse_and_late_weights(nf4, orc):
    """Random X within the fp32 bound; one workspace reused across calls; the
    late-weight-read mode (every read after griddepcontrol.wait) gives the same
    bits; classic split-K on the same workspace does not disturb later stream-K."""
    import torch
    M = 24
    probs, host = _multi_setup(nf4, M, "bf16", 77, sparse=False)
    ws = torch.zeros(nf4.nf4_gemm_multi_workspace_bytes(M, [h[3] for h in host], [h[4] for h in host]),
                     dtype=torch.uint8, device="cuda")
    a = [y.clone() for y in nf4.nf4_gemm_multi(probs, M=M, y_dtype="f32", workspace=ws)]
    # a classic split-K call writing its partials into the same buffer
    x, K, pk, am, d, N = probs[1]
    need = nf4.nf4_gemm_workspace_bytes(M, N, K, 4)
    big = torch.zeros(max(need, ws.numel()), dtype=torch.uint8, device="cuda")
    nf4.nf4_gemm(x, pk, am, d, N=N, K=K, y_dtype="f32", splits=4, workspace=big)
    b = [y.clone() for y in nf4.nf4_gemm_multi(probs, M=M, y_dtype="f32", workspace=big[:ws.numel()])]
    nf4.nf4_gemm_set_early_weight_reads(False)
    try:
        c = nf4.nf4_gemm_multi(probs, M=M, y_dtype="f32", workspace=ws)
    finally:
        nf4.nf4_gemm_set_early_weight_reads(True)
    torch.cuda.synchronize()
    for i, (x16, packed, kw, N, K) in enumerate(host):
        assert torch.equal(a[i].view(torch.int32), b[i].view(torch.int32)), i
        assert torch.equal(a[i].view(torch.int32), c[i].view(torch.int32)), i
        ref, mag = orc.gemm_reference(x16, orc.OUT_BF16, packed, N, K, 64, **kw)
        err = np.abs(a[i].cpu().numpy().astype(np.float64) - ref)
        assert (err <= K * 2.0 ** -23 * mag + 1e-30).all(), i
    assert int(ws.view(torch.int32)[:64].abs().sum()) == 0


def test_gemm_multi_many_problems_and_errors(nf4, orc):
    """56 problems (the size of an 8-layer step) in one launch, spot-checked; K=0
    gives Y=0; bad K and too many problems are rejected."""
    import torch
    M, K = 16, 512
    shapes = [(128 + 64 * (i % 3), K * (1 + i % 2), bool(i % 2)) for i in range(56)]
    probs, host = _multi_setup(nf4, M, "bf16", 5000, shapes)
    ys = nf4.nf4_gemm_multi(probs, M=M, y_dtype="f32")
    torch.cuda.synchronize()
    for i in (0, 1, 27, 55):
        x16, packed, kw, N, Ki = host[i]
        ref = _exact_reference(x16, "bf16", packed, N, Ki, 64, kw, orc)
        assert np.array_equal(_pos0(ys[i].cpu().numpy()), _pos0(ref.astype(np.float32))), i
    x, _, pk, a, d, N = probs[0]
    y0 = nf4.nf4_gemm_multi([(x, 0, pk, a, d, N)], M=M, y_dtype="f32")
    torch.cuda.synchronize()
    assert int(y0[0].abs().sum()) == 0
    with pytest.raises(nf4.NF4Error) as e:
        nf4.nf4_gemm_multi([(x, 96, pk, a, d, N)], M=M)
    assert e.value.status == 2
    with pytest.raises(nf4.NF4Error) as e:
        nf4.nf4_gemm_multi(probs + probs[:9], M=M)
    assert e.value.status == 2


@pytest.mark.parametrize("K", [64, 128, 256])
@pytest.mark.parametrize("M", [1, 16, 40])
def test_gemm_many_short_segments_per_cta(nf4, orc, M, K):
    """Small K (1-4 chunks per tile) and many tiles: every CTA's stream-K range
    holds several whole tiles, i.e. several short segments back to back, so the
    two TMEM accumulators are reused while earlier segments may still be in the
    MMA pipe.  Exact sums (sparse +-1 X) must come out bit for bit."""
    N = 128 * 148 * 4 + 64
    for dq in (False, True):
        packed, kw = _weights(N, K, 64, dq, seed=M * 7 + K + int(dq))
        x16 = _to16(_sparse_pm1(M, K, min(K, 64), M + K + 1), "bf16")
        ref = _exact_reference(x16, "bf16", packed, N, K, 64, kw, orc)
        for _ in range(2):
            y = _run(nf4, x16, "bf16", M, packed, kw, N, K, 64, "f32", 0).cpu().numpy()
            bad = _pos0(y) != _pos0(ref.astype(np.float32))
            assert not bad.any(), (M, K, dq, int(bad.sum()), np.argwhere(bad)[:3].tolist())


STRESS = [  # (M, N, K, blocksize): every token-tile width, ragged N and M, K from 1 chunk up
    (17, 1000, 192, 64), (33, 777, 320, 64), (65, 300, 448, 64), (129, 520, 640, 128), (257, 256, 256, 256),
    (300, 384, 128, 64), (3, 20000, 64, 64), (48, 9000, 128, 128), (100, 5000, 192, 64), (200, 2000, 4096, 4096),
]


@pytest.mark.parametrize("M,N,K,bs", STRESS)
def test_gemm_shape_stress_exact(nf4, orc, M, N, K, bs):
    """Odd shapes through stream-K, the classic split grid and nf4_gemm_multi:
    partial super-stages, ragged tiles, several token tiles, small and large K,
    general-blocksize scales -- Y exact (sparse +-1 X) in every mode."""
    import torch
    dq = (M + N) % 2 == 0
    packed, kw = _weights(N, K, bs, dq, seed=M * 31 + N + K)
    x16 = _to16(_sparse_pm1(M, K, min(K, 64), M * 3 + K), "bf16")
    ref = _pos0(_exact_reference(x16, "bf16", packed, N, K, bs, kw, orc).astype(np.float32))
    for splits in (0, 1, 3):
        y = _run(nf4, x16, "bf16", M, packed, kw, N, K, bs, "f32", splits).cpu().numpy()
        assert np.array_equal(_pos0(y), ref), (M, N, K, bs, splits)
    x = _x_tensor(x16, "bf16", M, K)
    if dq:
        prob = (x, K, dev(packed), None, nf4.DQ(dev(kw["qabsmax"]), dev(kw["code2"]), dev(kw["absmax2"]),
                                               kw["offset"]), N)
    else:
        prob = (x, K, dev(packed), dev(kw["absmax"]), None, N)
    ys = nf4.nf4_gemm_multi([prob, prob], M=M, blocksize=bs, y_dtype="f32")
    torch.cuda.synchronize()
    for y in ys:
        assert np.array_equal(_pos0(y.cpu().numpy()), ref), (M, N, K, bs, "multi")
