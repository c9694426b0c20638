"""Multi-process (N>1) host logic on CPU with the gloo backend, world size 2.

The path has no data-path collective: ranks only agree on the
timed-region maximum and the summed work.  These tests cover that reduction,
the per-rank work assignment (row shards / replicas) and the torchrun launch of
the reference arm.
"""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ms, b, e = bench.reduce_over_ranks(10.0 + 5 * rank, 1e9 * (rank + 1), 4e8 * (rank + 1), "cpu", world)
        # strong scaling: the ranks' row shards partition every weight exactly
        shards = bench.rank_tensors("cfg3", "strong", world, rank, layers=2)
        q.put((rank, ms, b, e, sum(t.n for t in shards), len(shards)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_reduction_and_shards():
    from synth import workloads as wl
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ms, b, e, n_shard, cnt in res:
        assert ms == 15.0                     # max over ranks
        assert b == 3e9 and e == 1.2e9        # sum over ranks
        assert cnt == 14
    full = sum(t.n for t in wl.config_tensors("cfg3", layers=2))
    assert sum(r[4] for r in res) == full     # row shards cover the model exactly once


def test_weak_scaling_assigns_full_set_per_rank():
    sys.path.insert(0, ROOT)
    import bench
    a = bench.rank_tensors("cfg2", "weak", 4, 0)
    b = bench.rank_tensors("cfg2", "weak", 4, 3)
    assert [t.n for t in a] == [t.n for t in b] and sum(t.n for t in a) == 25_598_361_600


def test_torchrun_reference_arm_rank0_only():
    """`bench.py --impl reference` under torchrun: rank 0 prints one JSON line,
    the other ranks exit 0 without work."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
           "--config", "cfg1", "--ref-step-seconds", "0.3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["cpu_baseline"]["kind"] == "oracle" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["n_gpus"] == 2


def test_bench_self_launches_n_ranks_dry_run():
    """`python bench.py --gpus 2` without torchrun re-launches itself on 2 local
    ranks (torch.distributed.run); --dry-run replaces the GPU work with a
    synthetic time (gloo), so the whole launch path runs here: exactly one JSON
    line, n_gpus 2, strong scaling whose row shards cover Qwen3-32B exactly once."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "2",
                        "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["config"]["key"] == "cfg3"
    assert d["config"]["elements_total"] == 31_205_621_760
    assert len(d["per_rank_ms_per_step"]) == 2
    # value = summed work over the slowest rank's time
    assert d["value"] == round(d["config"]["algorithmic_bytes_per_step_total"]
                               / (max(d["per_rank_ms_per_step"]) * 1e-3) / 1e9, 1)


def test_bench_world_size_mismatch_is_an_error():
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


def test_alg_bytes_match_store_formula():
    sys.path.insert(0, ROOT)
    import bench
    from synth import workloads as wl
    t = wl.config_tensors("cfg3")
    assert bench.alg_bytes_of(t, 64, True) == 78_509_261_824      # 78.51 GB per Qwen3 step
    t = wl.config_tensors("cfg1")
    assert bench.alg_bytes_of(t, 64, False) == 42_991_616


def test_shard_of_is_rank0_shard():
    sys.path.insert(0, ROOT)
    import bench
    from synth import workloads as wl
    a = bench.rank_tensors("cfg4", "strong", 1, 0, shard_of=8)
    b = wl.config_tensors("cfg4", world_size=8, rank=0)
    assert [(t.rows, t.cols) for t in a] == [(t.rows, t.cols) for t in b]
    assert sum(t.n for t in a) * 8 == 68_451_041_280
