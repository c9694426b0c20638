"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself.

Each test names what fixes the expected value: the paper / SPEC worked examples
(tests/golden/), closed forms, library conversions (torch CPU F16C, numpy,
ml_dtypes), a scipy re-derivation of the NF4 table, or brute force.  A
plausible mistake anywhere in the oracle -- a wrong table entry, swapped nibble
order, wrong scale index, fp64 instead of fp32 product, FMA in the DQ decode,
FTZ, wrong rounding -- fails at least one of them.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import ml_dtypes
import numpy as np
import pytest

from tests import npref
from synth import inputs as syn

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                yield [c.strip() for c in line.split("|")]


def _f32(s):
    s = s.strip()
    if s.lower().startswith("0x"):
        return np.array([int(s, 16)], np.uint32).view(np.float32)[0]
    return np.float32(float(s))


def _bits(x):
    return int(np.array([x], np.float32).view(np.uint32)[0])


# --------------------------------------------------------------------------
# codebook
# --------------------------------------------------------------------------
def test_codebook_rederived_from_qlora_quantiles(orc):
    """QLoRA create_normal_map(offset=0.9677083, use_extra_value=True): normal
    quantiles (scipy) over torch.linspace, sorted, divided by the max.  Must equal
    the oracle table bit for bit."""
    import scipy.stats as st
    import torch
    offset = 0.9677083
    v1 = st.norm.ppf(torch.linspace(offset, 0.5, 9)[:-1]).tolist()
    v3 = (-st.norm.ppf(torch.linspace(offset, 0.5, 8)[:-1])).tolist()
    values = torch.Tensor(v1 + [0] * (256 - 15) + v3).sort().values
    values /= values.max()
    uniq = np.unique(values.numpy())
    assert uniq.size == 16
    assert np.array_equal(uniq.view(np.uint32), orc.codebook().view(np.uint32))


def test_codebook_invariants_and_spec_values(orc):
    cb = orc.codebook()
    assert cb.dtype == np.float32 and cb.size == 16 and cb.nbytes == 64   # P:122 "64 bytes"
    assert np.all(np.diff(cb) > 0)                                       # S:33 strictly increasing
    assert _bits(cb[0]) == _bits(-1.0) and _bits(cb[15]) == _bits(1.0)
    assert _bits(cb[7]) == 0                                             # S:35 exact +0.0
    assert np.array_equal(cb, npref.NF4_DECIMAL.astype(np.float32))      # canonical decimals
    for kind, idx, val, cite in (l for l in _lines("spec_examples.txt") if l[0] == "codebook"):
        assert abs(float(cb[int(idx)]) - float(val)) <= 1e-7, cite


# --------------------------------------------------------------------------
# fp32 -> fp16 / bf16 round-to-nearest-even, exhaustive (readings R5, R6)
# --------------------------------------------------------------------------
def _exhaustive(orc, to_lib, to_oracle, dtype):
    chunk = 1 << 24

    def run(c):
        x = np.arange(c * chunk, (c + 1) * chunk, dtype=np.uint64).astype(np.uint32)
        got = to_oracle(x)
        ref = to_lib(x)
        ok = npref.same_bits(got, ref, dtype)
        return int((~ok).sum()), (x[~ok][:4].tolist() if not ok.all() else [])

    with ThreadPoolExecutor(8) as ex:
        res = list(ex.map(run, range((1 << 32) // chunk)))
    bad = sum(r[0] for r in res)
    assert bad == 0, [r[1] for r in res if r[0]][:3]


def test_f16_rne_exhaustive_vs_torch_cpu(orc):
    """All 2^32 fp32 bit patterns vs torch's CPU float->half (hardware F16C
    vcvtps2ph, round-to-nearest-even).  NaNs compared by class only (R9)."""
    import torch

    def lib(x):
        return torch.from_numpy(x.view(np.float32)).to(torch.float16).view(torch.int16).numpy().view(np.uint16)
    _exhaustive(orc, lib, orc.f32_to_f16_bits, "f16")


def test_f16_rne_sampled_vs_numpy(orc):
    """Second library: numpy.astype(float16) on 2^22 random patterns plus every
    pattern around the fp16 rounding boundaries of the normal/subnormal/overflow
    ranges."""
    rng = np.random.Generator(np.random.Philox(7))
    x = rng.integers(0, 1 << 32, 1 << 22, dtype=np.uint64).astype(np.uint32)
    edges = []
    for e in range(100, 144):                     # exponents from deep subnormal-fp16 to overflow
        base = np.uint32(e << 23)
        for mant in (0x0, 0x1000, 0x0FFF, 0x1001, 0x3000, 0x2000, 0x7FF000, 0x7FFFFF, 0x400000):
            for s in (0, 0x80000000):
                edges.append(int(base) | mant | s)
    x = np.concatenate([x, np.array(edges, np.uint32)])
    got = orc.f32_to_f16_bits(x)
    with np.errstate(over="ignore"):
        ref = x.view(np.float32).astype(np.float16).view(np.uint16)
    assert npref.same_bits(got, ref, "f16").all()


def test_bf16_rne_exhaustive_vs_ml_dtypes(orc):
    """All 2^32 fp32 bit patterns vs ml_dtypes.bfloat16 (RNE, no FTZ)."""
    def lib(x):
        return x.view(np.float32).astype(ml_dtypes.bfloat16).view(np.uint16)
    _exhaustive(orc, lib, orc.f32_to_bf16_bits, "bf16")


def test_rne_closed_forms(orc):
    # fp16: 65519.996 -> 65504 (7BFF), 65520 -> Inf
    assert orc.f32_to_f16_bits(np.array([_bits(65519.996)], np.uint32))[0] == 0x7BFF
    assert orc.f32_to_f16_bits(np.array([_bits(65520.0)], np.uint32))[0] == 0x7C00
    # smallest fp16 subnormal 2^-24; exactly 2^-25 ties to even (0); just above -> 2^-24
    assert orc.f32_to_f16_bits(np.array([_bits(2.0 ** -24)], np.uint32))[0] == 0x0001
    assert orc.f32_to_f16_bits(np.array([_bits(2.0 ** -25)], np.uint32))[0] == 0x0000
    assert orc.f32_to_f16_bits(np.array([_bits(2.0 ** -25) + 1], np.uint32))[0] == 0x0001
    # signed zero survives
    assert orc.f32_to_f16_bits(np.array([0x80000000], np.uint32))[0] == 0x8000
    assert orc.f32_to_bf16_bits(np.array([0x80000000], np.uint32))[0] == 0x8000
    # bf16 keeps fp32 subnormals (no FTZ): 1e-39 -> 0x000B
    assert orc.f32_to_bf16_bits(np.array([_bits(1e-39)], np.uint32))[0] == 0x000B


# --------------------------------------------------------------------------
# dequantization: worked examples, goldens, closed forms
# --------------------------------------------------------------------------
def _deq_byte(orc, byte, absmax, dtype):
    out = orc.dequantize(np.array([byte], np.uint8), 2, 64, orc.OUT_F16 if dtype == "f16" else orc.OUT_BF16,
                         absmax=np.array([absmax], np.float32))
    return [int(v) for v in out]


def test_spec_worked_examples(orc):
    for row in _lines("spec_examples.txt"):
        if row[0] == "dequant_byte":
            byte, am = row[1].split()
            f16, bf16 = [[int(h, 16) for h in s.split()] for s in row[2].split("/")]
            assert _deq_byte(orc, int(byte, 16), _f32(am), "f16") == f16, row[3]
            assert _deq_byte(orc, int(byte, 16), _f32(am), "bf16") == bf16, row[3]
        elif row[0] == "dequant_n":
            n, byte, am = row[1].split()
            f16, bf16 = [[int(h, 16) for h in s.split()] for s in row[2].split("/")]
            for dt, exp in ((orc.OUT_F16, f16), (orc.OUT_BF16, bf16)):
                out = orc.dequantize(np.array([int(byte, 16)], np.uint8), int(n), 64, dt,
                                     absmax=np.array([_f32(am)], np.float32))
                assert [int(v) for v in out] == exp, row[3]
        elif row[0] == "nibbles":
            packed = np.array([int(h, 16) for h in row[1].split()], np.uint8)
            want = [int(i) for i in row[2].split()]
            out = orc.dequantize(packed, len(want), 64, orc.OUT_F16, absmax=np.array([1.0], np.float32))
            cb16 = npref.to16(orc.codebook(), "f16")
            assert [int(v) for v in out] == [int(cb16[i]) for i in want], row[3]


def test_survey_goldens(orc):
    cb = npref.NF4_DECIMAL.astype(np.float32)
    for row in _lines("survey_goldens.txt"):
        if row[0] == "dq":
            c2, a2, off, a_bits, idx, dt, out_nf, out_fma = row[1:]
            c2, a2, off = (np.array([int(h, 16)], np.uint32).view(np.float32) for h in (c2, a2, off))
            # numpy re-derivation of the fixture: two separate float32 roundings
            a = ((c2 * a2).astype(np.float32) + off).astype(np.float32)
            assert int(a.view(np.uint32)[0]) == int(a_bits, 16)
            assert int(npref.to16(cb[int(idx)] * a, dt)[0]) == int(out_nf, 16)
            # the oracle through its DQ path must give the non-fused value
            dtc = orc.OUT_F16 if dt == "f16" else orc.OUT_BF16
            packed = np.array([(int(idx) << 4) | int(idx)], np.uint8)
            out = orc.dequantize(packed, 2, 64, dtc, qabsmax=np.array([0], np.uint8), code2=np.resize(c2, 256),
                                 absmax2=a2, offset=float(off[0]))
            assert int(out[0]) == int(out_nf, 16) != int(out_fma, 16)
            continue
        byte = int(row[0], 16)
        am = _f32(row[1])
        f16 = [int(h, 16) for h in row[2].split()]
        bf16 = [int(h, 16) for h in row[3].split()]
        p = np.array([cb[byte >> 4] * am, cb[byte & 15] * am], np.float32)
        assert npref.to16(p, "f16").tolist() == f16 and npref.to16(p, "bf16").tolist() == bf16
        assert _deq_byte(orc, byte, am, "f16") == f16
        assert _deq_byte(orc, byte, am, "bf16") == bf16


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_all_bytes_times_spec_scales(orc, dtype):
    """all 256 byte values x scales {0, 1, 0.5, 3.14159e-3, 6.5504e4}."""
    packed = np.arange(256, dtype=np.uint8)
    for s in (0.0, 1.0, 0.5, 3.14159e-3, 6.5504e4):
        absmax = np.full(8, s, np.float32)
        dt = orc.OUT_F16 if dtype == "f16" else orc.OUT_BF16
        got = orc.dequantize(packed, 512, 64, dt, absmax=absmax)
        ref = npref.dequant_np(packed, 512, 64, dtype, absmax=absmax)
        assert npref.same_bits(got, ref, dtype).all()


def test_unit_scale_gives_rounded_codebook(orc):
    """Closed form: absmax = 1.0 -> out[k] = RNE16(NF4[idx_k]) (SURVEY golden row 1)."""
    packed = np.array([0x01, 0x23, 0x45, 0x67, 0x89, 0xAB, 0xCD, 0xEF], np.uint8)
    f16 = orc.dequantize(packed, 16, 64, orc.OUT_F16, absmax=np.array([1.0], np.float32))
    bf16 = orc.dequantize(packed, 16, 64, orc.OUT_BF16, absmax=np.array([1.0], np.float32))
    assert [f"{v:04x}" for v in f16] == ("bc00 b992 b833 b652 b48d b1ea add4 0000 "
                                         "2d18 3126 33e0 3568 370d 3880 39c9 3c00").split()
    assert [f"{v:04x}" for v in bf16] == ("bf80 bf32 bf06 beca be92 be3d bdba 0000 "
                                          "3da3 3e25 3e7c 3ead 3ee2 3f10 3f39 3f80").split()


def test_signed_zero_and_subnormal_absmax(orc):
    # idx 0..6 with absmax +0 -> -0.0 (0x8000); idx 7..15 -> +0
    out = orc.dequantize(np.array([0x07, 0x8F], np.uint8), 4, 64, orc.OUT_F16, absmax=np.array([0.0], np.float32))
    assert out.tolist() == [0x8000, 0x0000, 0x0000, 0x0000]
    # subnormal absmax, bf16, no FTZ (item 10)
    out = orc.dequantize(np.array([0xFE], np.uint8), 2, 64, orc.OUT_BF16,
                         absmax=np.array([1e-39], np.float32))
    assert out.tolist() == [0x000B, 0x0008]


def test_power_of_two_scale_is_exact_scaling(orc):
    """S:206 linearity: absmax * 2^j scales every output by exactly 2^j (no overflow)."""
    packed = syn.random_codes(4096, 3)
    absmax = syn.hash_absmax(5, 0, 128)
    for dt, np16 in ((orc.OUT_F16, np.float16), (orc.OUT_BF16, ml_dtypes.bfloat16)):
        base = orc.dequantize(packed, 8192, 64, dt, absmax=absmax).view(np16).astype(np.float64)
        for j in (1, 3, -2):
            sc = orc.dequantize(packed, 8192, 64, dt, absmax=(absmax * np.float32(2.0 ** j)).astype(np.float32))
            sc = sc.view(np16).astype(np.float64)
            nz = np.abs(base) > 2.0 ** -10   # away from 16-bit subnormals where 2^j is not exact
            assert np.array_equal(sc[nz], base[nz] * 2.0 ** j)


def test_scale_locality(orc):
    """changing absmax[j] changes only elements [j*bs, (j+1)*bs)."""
    for bs in (64, 128):
        n = 64 * 1024
        packed = syn.random_codes(n // 2, 11)
        absmax = syn.hash_absmax(12, 0, n // bs)
        base = orc.dequantize(packed, n, bs, orc.OUT_F16, absmax=absmax)
        for j in (0, 7, n // bs - 1):
            a2 = absmax.copy()
            a2[j] *= np.float32(1.5)
            got = orc.dequantize(packed, n, bs, orc.OUT_F16, absmax=a2)
            diff = np.nonzero(got != base)[0]
            assert diff.size > 0 and diff.min() >= j * bs and diff.max() < (j + 1) * bs


def test_fp32_product_not_fp64(orc):
    """Reading R5 requires rounding the product to fp32 first.  Find inputs where a
    single rounding of the exact (fp64) product differs and check the oracle takes
    the fp32 route (closed form from numpy float32 vs float64 arithmetic)."""
    cb = npref.NF4_DECIMAL.astype(np.float32)
    scales = syn.hash_absmax(99, 0, 1 << 16)
    found = 0
    for s in scales:
        p32 = (cb * s).astype(np.float32)
        p64 = cb.astype(np.float64) * np.float64(s)
        d = np.nonzero(npref.to16(p32, "f16") != p64.astype(np.float16).view(np.uint16))[0]
        if d.size:
            i = int(d[0])
            packed = np.array([(i << 4) | i], np.uint8)
            out = orc.dequantize(packed, 2, 64, orc.OUT_F16, absmax=np.array([s], np.float32))
            assert int(out[0]) == int(npref.to16(p32[i:i + 1], "f16")[0])
            found += 1
            if found >= 5:
                break
    assert found >= 1


# --------------------------------------------------------------------------
# brute force on tiny inputs: tails, block sizes, ranges, both modes
# --------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("dq", [False, True])
def test_bruteforce_small_n(orc, dtype, dq):
    code2 = syn.dynamic_map_code2()
    dt = orc.OUT_F16 if dtype == "f16" else orc.OUT_BF16
    for n in list(range(1, 200)) + [511, 512, 513, 1023, 1024, 1025]:
        for bs in (64, 128, 256, 4096):
            seed = n * 7 + bs
            packed = syn.hash_packed(seed, 0, (n + 1) // 2)
            nb = -(-n // bs)
            if dq:
                kw = dict(qabsmax=syn.hash_qabsmax(seed, 0, nb), code2=code2,
                          absmax2=syn.hash_absmax2(seed, 0, -(-nb // 256)), offset=float(syn.hash_offset(seed)))
            else:
                kw = dict(absmax=syn.hash_absmax(seed, 0, nb))
            got = orc.dequantize(packed, n, bs, dt, **kw)
            ref = npref.dequant_np(packed, n, bs, dtype, **kw)
            assert npref.same_bits(got, ref, dtype).all(), (n, bs)


def test_dq_reduces_to_fp32_mode(orc):
    """Closed form (reading R7): absmax2 = 1, offset = 0 gives a = code2[q] exactly,
    so DQ output equals fp32-mode output with absmax[b] = code2[q[b]]."""
    code2 = syn.dynamic_map_code2()
    n, bs = 64 * 600, 64
    packed = syn.random_codes(n // 2, 5)
    q = syn.random_codes(n // bs, 6)
    ones = np.ones(-(-(n // bs) // 256), np.float32)
    dqo = orc.dequantize(packed, n, bs, orc.OUT_F16, qabsmax=q, code2=code2, absmax2=ones, offset=0.0)
    f32o = orc.dequantize(packed, n, bs, orc.OUT_F16, absmax=code2[q])
    assert np.array_equal(dqo, f32o)


def test_dq_group_index(orc):
    """absmax2 index is b // 256: changing absmax2[g] changes only blocks 256g..256g+255."""
    code2 = syn.dynamic_map_code2()
    n, bs = 64 * 1024, 64
    packed = syn.random_codes(n // 2, 8)
    q = syn.random_codes(n // bs, 9)
    a2 = syn.hash_absmax2(10, 0, 4)
    off = float(syn.hash_offset(10))
    base = orc.dequantize(packed, n, bs, orc.OUT_BF16, qabsmax=q, code2=code2, absmax2=a2, offset=off)
    a2b = a2.copy()
    a2b[2] *= np.float32(3.0)
    got = orc.dequantize(packed, n, bs, orc.OUT_BF16, qabsmax=q, code2=code2, absmax2=a2b, offset=off)
    d = np.nonzero(got != base)[0]
    assert d.min() >= 2 * 256 * bs and d.max() < 3 * 256 * bs


def test_ranges_and_threads_agree(orc):
    n, bs = 300001, 128
    packed = syn.hash_packed(1, 0, (n + 1) // 2)
    absmax = syn.hash_absmax(1, 0, -(-n // bs))
    full = orc.dequantize(packed, n, bs, orc.OUT_F16, absmax=absmax)
    thr = orc.dequantize(packed, n, bs, orc.OUT_F16, absmax=absmax, threads=8)
    part = orc.dequantize(packed, n, bs, orc.OUT_F16, absmax=absmax, k_begin=12345, k_end=200001)
    assert np.array_equal(full, thr)
    assert np.array_equal(full[12345:200001], part)


def test_invalid_arguments_rejected(orc):
    with pytest.raises(ValueError):
        orc.dequantize(np.zeros(1, np.uint8), 2, 64, orc.OUT_F16)  # neither absmax nor DQ
    with pytest.raises(ValueError):
        orc.dequantize(np.zeros(1, np.uint8), 2, 64, 7, absmax=np.ones(1, np.float32))


# --------------------------------------------------------------------------
# quantizer (input generator; readings R12, R13)
# --------------------------------------------------------------------------
def test_quantize_spec_examples(orc):
    cb = orc.codebook()
    cases = {
        "zeros64": np.zeros(64, np.float32),
        "twice_codebook_pad64": np.concatenate([2 * cb, np.zeros(48, np.float32)]).astype(np.float32),
        "single_minus3": np.array([-3.0], np.float32),
    }
    for row in (l for l in _lines("spec_examples.txt") if l[0] == "quantize"):
        packed, absmax = orc.quantize(cases[row[1]], 64)
        assert absmax[0] == np.float32(float(row[2])), row[4]
        want = bytes.fromhex(row[3])
        assert bytes(packed[:len(want)]) == want, row[4]


def test_quantize_thresholds_are_fp32_midpoints(orc):
    """Appendix A values; the 6 thresholds fl32 rounded up: x == t_i -> lower index,
    while exact-nearest would pick the upper."""
    t = orc.thresholds()
    cb = npref.NF4_DECIMAL
    mid = (cb[:-1] + cb[1:]) / 2
    assert np.array_equal(t, mid.astype(np.float32))
    rounded_up = sorted(int(i) for i in np.nonzero(t.astype(np.float64) > mid)[0])
    assert rounded_up == [0, 1, 3, 4, 12, 14]
    # x exactly at each threshold with absmax 1 (x = 1.0 element fixes absmax)
    for i in range(15):
        x = np.array([1.0, t[i]], np.float32)
        packed, _ = orc.quantize(x, 64)
        assert (packed[0] & 0x0F) == i   # strict '>' -> lower code i


def test_quantize_codebook_roundtrip_many_scales(orc):
    """x = fl32(s * c_i) must quantize to code i (SURVEY item 15)."""
    cb = orc.codebook()
    rng = np.random.Generator(np.random.Philox(3))
    scales = np.concatenate([10 ** rng.uniform(-4, 3, 4000), [1, 2, 0.5, 3, 1e-30, 65504]]).astype(np.float32)
    x = (scales[:, None] * cb[None, :]).astype(np.float32)      # 16 values per row
    x = np.concatenate([x, np.zeros((x.shape[0], 48), np.float32)], axis=1).reshape(-1)
    packed, absmax = orc.quantize(x, 64)
    assert np.array_equal(absmax, scales)
    idx = np.stack([packed.reshape(-1, 32)[:, :8] >> 4, packed.reshape(-1, 32)[:, :8] & 15], -1).reshape(-1, 16)
    assert (idx == np.arange(16)).all()


def test_quantize_error_bound_and_idempotence(orc):
    """|x - xhat| <= 0.1519036 * absmax (half the max code gap c1 - c0; SURVEY
    item 17 corrects S:124) and quantize(dequantize(quantize(x))) is a fixed point
    (S:125).  xhat here is the fp32 product (numpy)."""
    cb = npref.NF4_DECIMAL.astype(np.float32)
    half_gap = (cb[1] - cb[0]) / 2
    assert abs(float(half_gap) - 0.1519036) < 1e-6
    x = syn.gaussian_weights(1 << 20, 4, std=1.0)
    packed, absmax = orc.quantize(x, 64)
    k = np.arange(x.size)
    idx = np.where(k % 2 == 0, packed[k >> 1] >> 4, packed[k >> 1] & 15)
    xhat = (cb[idx] * absmax[k // 64]).astype(np.float32)
    err = np.abs(x.astype(np.float64) - xhat) / absmax[k // 64]
    assert err.max() <= 0.1519036 + 1e-6
    p2, a2 = orc.quantize(xhat, 64)
    assert np.array_equal(p2, packed) and np.array_equal(a2, absmax)


def test_quantize_matches_nearest_code_except_ties(orc):
    """Away from the 15 thresholds the threshold rule equals the exact argmin
    over the 16 codes."""
    cb64 = npref.NF4_DECIMAL
    x = syn.gaussian_weights(64 * 4096, 21, std=1.0)
    packed, absmax = orc.quantize(x, 64)
    k = np.arange(x.size)
    idx = np.where(k % 2 == 0, packed[k >> 1] >> 4, packed[k >> 1] & 15)
    xn = (x * (np.float32(1.0) / absmax[k // 64])).astype(np.float32).astype(np.float64)
    nearest = np.argmin(np.abs(xn[:, None] - cb64[None, :]), axis=1)
    assert np.array_equal(idx, nearest)


def test_quantize_odd_tail_pad_nibble(orc):
    x = syn.gaussian_weights(129, 2)
    packed, absmax = orc.quantize(x, 64)
    assert packed.size == 65 and absmax.size == 3 and (packed[-1] & 0x0F) == 0


def test_double_quantize_bruteforce(orc):
    """Second level: d = fl32(a - offset), s2 = max|d| per 256, dn = fl32(d * fl32(1/s2)),
    q = argmin fl32|dn - code2[i]| (ties -> lowest); checked with numpy brute force."""
    code2 = syn.dynamic_map_code2()
    absmax = syn.hash_absmax(33, 0, 256 * 5 + 17)
    off = np.float32(absmax.astype(np.float64).mean())
    q, a2 = orc.double_quantize(absmax, float(off), code2, 256)
    d = (absmax - off).astype(np.float32)
    for g in range(a2.size):
        dg = d[g * 256:(g + 1) * 256]
        s2 = np.abs(dg).max()
        assert a2[g] == s2
        dn = (dg * (np.float32(1.0) / s2)).astype(np.float32)
        dist = np.abs((dn[:, None] - code2[None, :]).astype(np.float32))
        assert np.array_equal(q[g * 256:(g + 1) * 256], np.argmin(dist, axis=1))
    # decoded absmax stays close to the original (8-bit dynamic code, |dn| <= 1)
    t = (code2[q] * a2[np.arange(absmax.size) // 256]).astype(np.float32)
    dec = (t + off).astype(np.float32)
    assert np.max(np.abs(dec - absmax) / np.abs(absmax)) < 0.05


def dq_tie_fixture():
    """Blocks whose normalized second-level value dn sits EXACTLY midway between
    two adjacent code2 entries (fl32|dn - c_i| == fl32|dn - c_i+1|), so the
    tie rule alone decides q.  Group 0: offset 0, one block at absmax 1.0 makes
    s2 = 1 and dn = absmax exactly; group 1 (second call) uses offset 1.0 and a
    block at 2.0 (d = +1) so d = absmax - 1 reaches the negative midpoints.
    Returns [(absmax fp32[256], offset, expected q per tie block {block: i})]."""
    code2 = syn.dynamic_map_code2()
    ties = []
    for i in range(255):
        m = (np.float64(code2[i]) + np.float64(code2[i + 1])) / 2
        if np.float64(np.float32(m)) != m:
            continue
        m32 = np.float32(m)
        if abs(np.float32(m32 - code2[i])) == abs(np.float32(m32 - code2[i + 1])):
            ties.append((i, m32))
    assert len(ties) > 100
    out = []
    # non-negative midpoints, offset 0
    pos = [(i, m) for i, m in ties if m >= 0][:200]
    a = np.full(256, 0.5, np.float32)
    a[0] = 1.0
    exp = {}
    for j, (i, m) in enumerate(pos[:255]):
        a[1 + j] = m
        exp[1 + j] = i
    out.append((a, 0.0, exp))
    # negative midpoints through offset 1.0: absmax = 1 + m must give d = m exactly
    neg = [(i, m) for i, m in ties if m < 0 and np.float32(np.float32(1.0 + m) - np.float32(1.0)) == m]
    a = np.full(256, 1.0, np.float32)
    a[0] = 2.0
    exp = {}
    for j, (i, m) in enumerate(neg[:255]):
        a[1 + j] = np.float32(1.0 + m)
        exp[1 + j] = i
    assert len(exp) > 20
    out.append((a, 1.0, exp))
    return code2, out


def test_double_quantize_ties_go_to_lower_index(orc):
    """SPEC S:98 / S:129 (nearest code, ties broken toward the smaller index;
    SURVEY 8(c) item 19): every exact tie must choose the LOWER code2 index.
    Expected indices come from the fixture's construction (i, not i + 1), not
    from any implementation."""
    code2, cases = dq_tie_fixture()
    for absmax, off, exp in cases:
        q, a2 = orc.double_quantize(absmax, off, code2, 256)
        assert a2[0] == 1.0
        for b, i in exp.items():
            assert q[b] == i, (b, i, int(q[b]), float(absmax[b]))


def test_double_quantize_zero_group(orc):
    code2 = syn.dynamic_map_code2()
    absmax = np.full(300, 0.25, np.float32)
    q, a2 = orc.double_quantize(absmax, 0.25, code2, 256)
    assert (a2 == 0).all() and (code2[q] == 0).all()


# --------------------------------------------------------------------------
# other 16-entry codebooks and fp32 output
# --------------------------------------------------------------------------
def test_explicit_nf4_codebook_is_default(orc):
    packed = syn.random_codes(5000, 1)
    absmax = syn.hash_absmax(2, 0, 10000 // 64 + 1)
    a = orc.dequantize(packed, 10000, 64, orc.OUT_BF16, absmax=absmax)
    b = orc.dequantize(packed, 10000, 64, orc.OUT_BF16, absmax=absmax, codebook=orc.codebook())
    assert np.array_equal(a, b)


def test_fp32_output_is_the_fp32_product(orc):
    """OUT_F32 returns fl32(CB[idx] * a) itself (numpy float32 multiply), both modes."""
    code2 = syn.dynamic_map_code2()
    for dq in (False, True):
        for n in (1, 2, 63, 1025, 70001):
            packed = syn.hash_packed(n, 0, (n + 1) // 2)
            nb = -(-n // 64)
            kw = (dict(qabsmax=syn.hash_qabsmax(n, 0, nb), code2=code2, absmax2=syn.hash_absmax2(n, 0, -(-nb // 256)),
                       offset=float(syn.hash_offset(n))) if dq else dict(absmax=syn.hash_absmax(n, 0, nb)))
            got = orc.dequantize(packed, n, 64, orc.OUT_F32, **kw)
            assert np.array_equal(got, npref.dequant_np(packed, n, 64, "f32", **kw))


def test_fp4_table_closed_forms(orc):
    """BNB FP4 table with absmax 1: fp32 output is the table exactly; 16-bit
    outputs are its RNE roundings (numpy / ml_dtypes)."""
    cb = syn.bnb_fp4_codebook()
    assert cb[3] == 1.0 and cb[11] == -1.0 and cb[0] == 0 and np.signbit(cb[8])
    packed = np.array([0x01, 0x23, 0x45, 0x67, 0x89, 0xAB, 0xCD, 0xEF], np.uint8)
    one = np.array([1.0], np.float32)
    f32 = orc.dequantize(packed, 16, 64, orc.OUT_F32, absmax=one, codebook=cb)
    assert np.array_equal(f32, cb.view(np.uint32))
    for dt, code in (("f16", orc.OUT_F16), ("bf16", orc.OUT_BF16)):
        got = orc.dequantize(packed, 16, 64, code, absmax=one, codebook=cb)
        assert np.array_equal(got, npref.to16(cb, dt))


@pytest.mark.parametrize("dtype", ["f16", "bf16", "f32"])
def test_custom_codebook_bruteforce(orc, dtype):
    rng = np.random.Generator(np.random.Philox(9))
    cb = rng.standard_normal(16).astype(np.float32)
    code = {"f16": orc.OUT_F16, "bf16": orc.OUT_BF16, "f32": orc.OUT_F32}[dtype]
    for n in (1, 17, 1000, 4097):
        packed = syn.hash_packed(n + 5, 0, (n + 1) // 2)
        absmax = syn.hash_absmax(n + 5, 0, -(-n // 128))
        got = orc.dequantize(packed, n, 128, code, absmax=absmax, codebook=cb)
        assert np.array_equal(got, npref.dequant_np(packed, n, 128, dtype, absmax=absmax, codebook=cb))


# --------------------------------------------------------------------------
# F1 reference (oracle.gemm_reference): Y = X . W^T over the oracle's weights
# --------------------------------------------------------------------------
def _codebook_rows(N, K):
    """Row n holds codes (n + k) mod 16 (high nibble first); absmax 1.0 everywhere."""
    codes = (np.arange(N)[:, None] + np.arange(K)[None, :]) % 16
    flat = codes.reshape(-1).astype(np.uint8)
    return (flat[0::2] << 4 | flat[1::2]).astype(np.uint8), codes


@pytest.mark.parametrize("x_dtype", ["bf16", "f16"])
def test_gemm_reference_one_hot_and_ones(orc, x_dtype):
    """Closed forms independent of the oracle's C: with absmax 1 every weight is
    RNE16(NF4[code]) (ml_dtypes / numpy rounding of the pinned table), so a one-hot
    row of X returns one weight and an all-ones row returns the row sum."""
    N, K = 5, 128
    packed, codes = _codebook_rows(N, K)
    absmax = np.ones(N * K // 64, np.float32)
    np16 = ml_dtypes.bfloat16 if x_dtype == "bf16" else np.float16
    code = orc.OUT_BF16 if x_dtype == "bf16" else orc.OUT_F16
    w = orc.codebook().astype(np16).astype(np.float64)[codes]          # [N, K]
    ks = np.array([0, 7, 64, 127])
    x = np.zeros((len(ks) + 1, K), np.float32)
    x[np.arange(len(ks)), ks] = 1.0
    x[-1, :] = 1.0
    x16 = x.astype(np16).view(np.uint16)
    y, s = orc.gemm_reference(x16, code, packed, N, K, 64, absmax=absmax)
    assert np.array_equal(y[:-1], w[:, ks].T)
    assert np.array_equal(y[-1], w.sum(axis=1))
    assert np.array_equal(s[-1], np.abs(w).sum(axis=1))


def test_gemm_reference_linearity_and_magnitude(orc):
    """Integer-valued X keeps every fp64 product and sum exact (|values| < 2^53), so
    the reference must be exactly linear in X; S = |X|.|W|^T bounds |Y| and equals
    Y for non-negative X and W."""
    N, K = 6, 256
    packed = syn.hash_packed(41, 0, N * K // 2)
    absmax = np.full(N * K // 64, 2.0, np.float32)
    rng = np.random.default_rng(5)
    x1 = rng.integers(-8, 9, (3, K)).astype(np.float32)
    x2 = rng.integers(-8, 9, (3, K)).astype(np.float32)
    b = lambda a: a.astype(ml_dtypes.bfloat16).view(np.uint16)       # noqa: E731 (exact for |v| <= 256)
    y1, s1 = orc.gemm_reference(b(x1), orc.OUT_BF16, packed, N, K, 64, absmax=absmax)
    y2, _ = orc.gemm_reference(b(x2), orc.OUT_BF16, packed, N, K, 64, absmax=absmax)
    y12, _ = orc.gemm_reference(b(x1 + x2), orc.OUT_BF16, packed, N, K, 64, absmax=absmax)
    assert np.array_equal(y12, y1 + y2)
    assert (np.abs(y1) <= s1).all()
    # non-negative weights: codes 8..15 only (NF4 >= 0 there), non-negative X -> S == Y
    pos = (syn.hash_packed(42, 0, N * K // 2) | 0x88).astype(np.uint8)
    yp, sp = orc.gemm_reference(b(np.abs(x1)), orc.OUT_BF16, pos, N, K, 64, absmax=absmax)
    assert np.array_equal(yp, sp)


def test_oracle_memory_safe_under_asan_ubsan(tmp_path):
    """the oracle built with -fsanitize=address,undefined, driven over
    n = 1..1100 x blocksizes x modes x output types with exactly-sized buffers
    and sub-range calls (tests/oracle_asan_driver.c): no sanitizer report, and
    sub-range results equal the full-range result."""
    import subprocess
    here = os.path.dirname(os.path.abspath(__file__))
    src = os.path.join(os.path.dirname(here), "oracle", "oracle.c")
    exe = tmp_path / "oracle_asan"
    cc = ["gcc", "-O1", "-g", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fsanitize=address,undefined",
          "-fno-sanitize-recover=all", "-o", str(exe), src, os.path.join(here, "oracle_asan_driver.c")]
    r = subprocess.run(cc, capture_output=True, text=True)
    if r.returncode != 0 and "sanitize" in r.stderr:
        pytest.skip("gcc sanitizer runtime unavailable: " + r.stderr[-200:])
    assert r.returncode == 0, r.stderr[-2000:]
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=1"))
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    assert "0 failures" in r.stdout
