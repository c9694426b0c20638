"""Workload shapes (synth/workloads.py) against the model sizes they encode."""
from __future__ import annotations

import pytest

from synth import workloads as wl


@pytest.mark.parametrize("model,total", [("gemma-3-27b", 25_598_361_600), ("qwen3-32b", 31_205_621_760),
                                         ("llama-3.3-70b", 68_451_041_280)])
def test_model_totals(model, total):
    """SURVEY 8(d) element totals; Qwen3-32B has 64 layers."""
    ts = wl.model_tensors(model)
    assert sum(t.n for t in ts) == total
    assert len(ts) == 7 * wl.MODELS[model][0]
    if model == "qwen3-32b":
        assert wl.MODELS[model][0] == 64


@pytest.mark.parametrize("model", sorted(wl.MODELS))
@pytest.mark.parametrize("g", [1, 2, 4, 8])
def test_shards_multiple_of_16384(model, g):
    """Every row shard is a multiple of 64*256 elements: shard boundaries align with
    both quantization levels and with the kernel's 16384-element tile."""
    for t in wl.model_tensors(model, layers=1, world_size=g, rank=g - 1):
        assert t.n % 16384 == 0


def test_algorithmic_bytes_per_element():
    assert wl.algorithmic_bytes_per_element(64, False) == 2.5625
    assert abs(wl.algorithmic_bytes_per_element(64, True) - 2.515869140625) < 1e-12
    assert abs(wl.algorithmic_bytes_per_element(4096, True) - 2.500248) < 1e-6


def test_weight_store_bytes_match_formula():
    """WeightStore.algorithmic_bytes (bench numerator) == per-element formula x n
    for whole-block tensors (+1 KB code2 per pass in DQ mode)."""
    from paper_2604_02556_b200.weights import Entry, WeightStore
    ws = WeightStore(64, True, "bf16")
    ws.entries = [Entry("a", 4096 * 5376, 0, 0, 0, 0, 0)]
    n = 4096 * 5376
    assert ws.algorithmic_bytes() == n // 2 + 2 * n + n // 64 + 4 * (n // 64 // 256) + 1024
    ws.dq = False
    assert ws.algorithmic_bytes() == n // 2 + 2 * n + 4 * (n // 64)
