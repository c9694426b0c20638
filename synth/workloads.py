"""Workload shapes: the paper's three models and BASELINE.json's configs.

"All linear weights" = the 7 decoder-layer projections (q, k, v, o, gate, up,
down).  lm_head and embeddings are not quantized (HF's BnB skip list).
Shapes are [out_features, in_features] from the public model configs ([ext];
the Qwen3-32B layer count 64 matches P:60).  Every tensor size and every
row-shard for G in {1,2,4,8} is a multiple of 16384 = 64 * 256 (checked in
tests/test_workloads.py).
"""
from __future__ import annotations

from dataclasses import dataclass

MODELS = {
    "gemma-3-27b": (62, [(4096, 5376), (2048, 5376), (2048, 5376), (5376, 4096),
                         (21504, 5376), (21504, 5376), (5376, 21504)]),
    "qwen3-32b": (64, [(8192, 5120), (1024, 5120), (1024, 5120), (5120, 8192),
                       (25600, 5120), (25600, 5120), (5120, 25600)]),
    "llama-3.3-70b": (80, [(8192, 8192), (1024, 8192), (1024, 8192), (8192, 8192),
                           (28672, 8192), (28672, 8192), (8192, 28672)]),
}
PROJ = ["q_proj", "k_proj", "v_proj", "o_proj", "gate_proj", "up_proj", "down_proj"]


@dataclass(frozen=True)
class Tensor:
    name: str
    rows: int
    cols: int

    @property
    def n(self) -> int:
        return self.rows * self.cols


def model_tensors(model: str, layers: int | None = None, world_size: int = 1, rank: int = 0):
    """The linear weights of ``model`` (optionally the first ``layers`` layers),
    each row-sharded ``world_size`` ways; returns rank ``rank``'s shards."""
    n_layers, shapes = MODELS[model]
    if layers is not None:
        n_layers = min(n_layers, layers)
    out = []
    for layer in range(n_layers):
        for pname, (rows, cols) in zip(PROJ, shapes):
            assert rows % world_size == 0
            r = rows // world_size
            out.append(Tensor(f"layers.{layer}.{pname}[{rank}/{world_size}]", r, cols))
    return out


@dataclass(frozen=True)
class Config:
    key: str
    description: str
    model: str | None
    blocksize: int
    dq: bool
    out_dtype: str  # "f16" | "bf16"


CONFIGS = {
    "cfg1": Config("cfg1", "single 4096x4096 NF4 weight, blocksize 64, fp32 absmax, fp16 output",
                   None, 64, False, "f16"),
    "cfg2": Config("cfg2", "Gemma-27B linear-layer set, blocksize 64, double-quant absmax, bf16 output",
                   "gemma-3-27b", 64, True, "bf16"),
    "cfg3": Config("cfg3", "Qwen3-32B all linear weights, blocksize 64, double-quant, fp16 output",
                   "qwen3-32b", 64, True, "f16"),
    "cfg4": Config("cfg4", "Llama-3.3-70B all linear weights, row-sharded, double-quant, bf16 output",
                   "llama-3.3-70b", 64, True, "bf16"),
}


def config_tensors(key: str, world_size: int = 1, rank: int = 0, layers: int | None = None):
    cfg = CONFIGS[key]
    if cfg.model is None:
        return [Tensor("w[4096x4096]", 4096, 4096)]
    return model_tensors(cfg.model, layers=layers, world_size=world_size, rank=rank)


def algorithmic_bytes_per_element(blocksize: int, dq: bool, blocksize2: int = 256) -> float:
    """codes 0.5 B + absmax per block + 2 B output per element."""
    if dq:
        return 0.5 + 1.0 / blocksize + 4.0 / (blocksize2 * blocksize) + 2.0
    return 0.5 + 4.0 / blocksize + 2.0
