"""NF4Linear (paper_2604_02556_b200/nn.py): GPU quantization -> storage -> forward.

The stored weight is the oracle's quantization of the same input (F2, bit-exact),
dequantize() is the hot path (bit-exact), and forward() matches X.W^T within the
fp32-accumulation bound for both the fused (decode) and the dequantize+GEMM
(prefill) paths."""
from __future__ import annotations

import ml_dtypes
import numpy as np
import pytest

from synth import inputs as syn

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nn():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_02556_b200 import nn as m
    return m


@pytest.mark.parametrize("dq", [True, False])
def test_nf4linear_matches_oracle(nn, orc, dq):
    import torch
    out_f, in_f = 384, 1024
    w = syn.gaussian_weights(out_f * in_f, 5).reshape(out_f, in_f)
    lin = nn.NF4Linear.from_weight(torch.from_numpy(w).cuda(), double_quant=dq)
    packed, absmax = orc.quantize(w.reshape(-1), 64)
    assert np.array_equal(lin.packed.cpu().numpy(), packed)
    if dq:
        code2 = syn.dynamic_map_code2()
        q, a2 = orc.double_quantize(absmax, lin.offset, code2)
        assert np.array_equal(lin.qabsmax.cpu().numpy(), q) and np.array_equal(lin.absmax2.cpu().numpy(), a2)
        kw = dict(qabsmax=q, code2=code2, absmax2=a2, offset=lin.offset)
    else:
        assert np.array_equal(lin.absmax.cpu().numpy(), absmax)
        kw = dict(absmax=absmax)
    wdeq = orc.dequantize(packed, out_f * in_f, 64, orc.OUT_BF16, **kw)
    got = lin.dequantize().view(torch.int16).cpu().numpy().view(np.uint16).reshape(-1)
    assert np.array_equal(got, wdeq)
    wd = wdeq.view(ml_dtypes.bfloat16).astype(np.float64).reshape(out_f, in_f)
    for M in (3, 64, 200):                     # fused path, fused path, dequantize + GEMM path
        x = syn.gaussian_weights(M * in_f, M, std=1.0).reshape(M, in_f)
        xb = x.astype(ml_dtypes.bfloat16)
        y = lin(torch.from_numpy(xb.view(np.uint16).view(np.int16)).view(torch.bfloat16).cuda().reshape(1, M, in_f))
        assert y.shape == (1, M, out_f)
        y = y.float().cpu().numpy().reshape(M, out_f).astype(np.float64)
        xd = xb.astype(np.float64)
        ref, mag = xd @ wd.T, np.abs(xd) @ np.abs(wd).T
        bound = in_f * 2.0 ** -23 * mag * (1 + 2.0 ** -8) + np.abs(ref) * 2.0 ** -8 + 1e-30
        assert (np.abs(y - ref) <= bound).all(), M


def test_nf4lineargroup_matches_members(nn):
    """NF4LinearGroup (one grouped launch) agrees with each member's own forward
    within the fp32 accumulation bound, and falls back for prefill-size M."""
    import torch
    in_f = 1024
    lins = []
    for i, out_f in enumerate((512, 256, 256)):
        w = syn.gaussian_weights(out_f * in_f, 20 + i).reshape(out_f, in_f)
        lins.append(nn.NF4Linear.from_weight(torch.from_numpy(w).cuda(), double_quant=(i != 1)))
    grp = nn.NF4LinearGroup(lins)
    for M in (1, 16, 200, 300):
        x = torch.from_numpy(syn.gaussian_weights(M * in_f, 7 + M, std=1.0).reshape(M, in_f)).cuda().to(torch.bfloat16)
        outs = grp(x)
        for lin, y in zip(lins, outs):
            wd = lin.dequantize().float().double()
            xd = x.double()
            ref, mag = xd @ wd.T, xd.abs() @ wd.abs().T
            bound = in_f * 2.0 ** -23 * mag * (1 + 2.0 ** -8) + ref.abs() * 2.0 ** -8 + 1e-30
            assert ((y.double() - ref).abs() <= bound).all(), M


def test_nf4linear_state_dict_round_trip_keeps_offset_and_bias():
    """the double-quant offset and the bias are module state; a
    save/load round trip into a fresh layer gives identical outputs."""
    import io
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_02556_b200.nn import NF4Linear
    torch.manual_seed(0)
    w = torch.randn(384, 512, device="cuda") * 0.02
    b = torch.randn(384, device="cuda")
    a = NF4Linear.from_weight(w, bias=b)
    assert a.offset != 0.0
    buf = io.BytesIO()
    torch.save(a.state_dict(), buf)
    buf.seek(0)
    fresh = NF4Linear(512, 384, bias=True, device="cuda")
    fresh.load_state_dict(torch.load(buf))
    assert fresh.offset == a.offset
    x = torch.randn(8, 512, device="cuda", dtype=torch.bfloat16)
    assert torch.equal(a(x), fresh(x))
    assert torch.equal(a.dequantize(), fresh.dequantize())
