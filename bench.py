#!/usr/bin/env python
"""Benchmark: blockwise NF4 dequantization on B200 (arxiv 2604.02556 hot path).

A *step* is one pass of the whole hot path over a model's NF4 linear weights
(all 7 projections of every decoder layer) -- what one inference forward
pass dequantizes.  Default workload: BASELINE.json configs[2], the Qwen3-32B
linear weights (the paper's profiled model, Table I), blocksize 64,
double-quantized absmax, fp16 output (the paper's output type): 31.2 G
elements, 78.5 GB of algorithmic traffic per step at N=1 -- the largest
configuration that fits one GPU and the one the metric's "1/2/4/8 GPUs" is
quoted on.  Inputs and outputs are far larger than the 126 MB L2, so no flush
is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3]
                    [--inputs gaussian|hash] [--scaling strong|weak] [--impl ours|reference]

Multi-GPU: one process per GPU.  Under torchrun (the driver) RANK/WORLD_SIZE come
from the environment and must match --gpus; without torchrun, `--gpus N` > 1
re-launches itself through torch.distributed.run on N local ranks.  The path has
no exchange step, so there is no data-path collective: with
--scaling strong (default) every weight is row-sharded N ways and each rank
quantizes and dequantizes its own shards (what an N-GPU tensor-parallel
deployment holds); --scaling weak gives every rank a full model replica.  Time
is measured with CUDA events on the launching stream, max over ranks; NCCL
carries only the barrier and that max.

Rank 0 prints ONE JSON line: `value` = whole-job algorithmic GB/s (SURVEY 8(d):
codes ceil(n/2) + scales + 2 B/elt output), `e2e` the same metric through the
host-buffer C-ABI call (pinned host -> HBM -> host, copies timed), `roofline`
the dequant kernel against the measured HBM copy peak (from the timed pass),
`cpu_baseline` the CPU oracle on a bounded sample on this host's cores (all
threads and one thread), `extra_configs` the same step on config 2 (Gemma-3-27B,
bf16) and config 1 (one 4096x4096 tensor: L2-resident, so timed over rotating
cold copies launched from one CUDA graph), and `f1` the fused NF4 dequant +
tcgen05 GEMM over 8 Gemma-3-27B decoder layers at M = 1 / 16 /
64 tokens.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from synth import inputs as syn  # noqa: E402
from synth import workloads as wl  # noqa: E402

METRIC = "NF4 dequant HBM GB/s & % of B200 peak, Gelem/s at 1/2/4/8 GPUs"
UNIT = "GB/s"
NOMINAL_HBM_GBS = 8000.0


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, smax, power, reasons = [], 0.0, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = max(smax, float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power) if power else None}


# ---------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline and the --impl reference arm)
# ---------------------------------------------------------------------------
def oracle_sample_inputs(cfg, n):
    """Counter-based inputs for the first n elements of a tensor of the workload."""
    from synth import fast
    c = wl.CONFIGS[cfg]
    bs = c.blocksize
    nb = -(-n // bs)
    packed = fast.packed(7, 0, (n + 1) // 2)
    if c.dq:
        kw = dict(qabsmax=fast.qabsmax(7, 0, nb), code2=syn.dynamic_map_code2(),
                  absmax2=fast.absmax2(7, 0, -(-nb // 256)), offset=float(syn.hash_offset(7)))
    else:
        kw = dict(absmax=fast.absmax(7, 0, nb))
    return packed, kw


_SAMPLE_CACHE = {}


def _sample(cfg, n):
    """Counter-based inputs for a sample of n elements, generated once per (cfg, n)."""
    key = (cfg, n)
    if key not in _SAMPLE_CACHE:
        _SAMPLE_CACHE.clear()
        _SAMPLE_CACHE[key] = oracle_sample_inputs(cfg, n)
    return _SAMPLE_CACHE[key]


def size_oracle_sample(cfg, target_s, threads):
    """Elements the oracle processes in ~target_s seconds on `threads` threads."""
    import oracle
    c = wl.CONFIGS[cfg]
    code = oracle.OUT_F16 if c.out_dtype == "f16" else oracle.OUT_BF16
    probe_n = (1 << 25) if threads > 1 else (1 << 23)   # larger than the host caches, like the sample
    packed, kw = oracle_sample_inputs(cfg, probe_n)
    oracle.dequantize(packed, 1 << 20, c.blocksize, code, threads=threads, **kw)   # load + warm up
    t0 = time.perf_counter()
    oracle.dequantize(packed, probe_n, c.blocksize, code, threads=threads, **kw)
    rate = probe_n / max(time.perf_counter() - t0, 1e-6)
    n = max(1 << 22, min(int(rate * target_s), 1 << 31))
    return n - n % 16384


def time_oracle(cfg, target_s=10.0, threads=None, n=None):
    """Time the oracle (as it stands) on this host's cores over a bounded sample
    of the workload (~target_s seconds, or exactly n elements).  Returns a
    cpu_baseline dict."""
    import oracle
    c = wl.CONFIGS[cfg]
    threads = threads or len(os.sched_getaffinity(0))
    code = oracle.OUT_F16 if c.out_dtype == "f16" else oracle.OUT_BF16
    resize = n is None
    if n is None:
        n = size_oracle_sample(cfg, target_s, threads)
    while True:
        packed, kw = _sample(cfg, n)
        t0 = time.perf_counter()
        oracle.dequantize(packed, n, c.blocksize, code, threads=threads, **kw)
        dt = time.perf_counter() - t0
        if not resize or dt >= 0.5 * target_s or n >= 1 << 31:
            break
        resize = False                      # one re-size from a full-size run
        n = int(min(1 << 31, n * target_s / max(dt, 1e-3)))
        n -= n % 16384
    passes = 1
    if resize and n >= 1 << 31 and dt < 0.5 * target_s:
        # the sample is capped at 2^31 elements (host RAM); repeat it to reach ~target_s of CPU work
        passes = max(1, int(round(target_s / max(dt, 1e-3))))
        t0 = time.perf_counter()
        for _ in range(passes):
            oracle.dequantize(packed, n, c.blocksize, code, threads=threads, **kw)
        dt = time.perf_counter() - t0
    bpe = wl.algorithmic_bytes_per_element(c.blocksize, c.dq)
    total = n * passes
    return {"value": round(total * bpe / dt / 1e9, 3), "unit": UNIT, "cores": threads, "kind": "oracle",
            "gelem_per_s": round(total / dt / 1e9, 4), "seconds": round(dt, 2), "elements": n,
            "sample": f"one synthetic tensor of {n} elements"
                      + (f" dequantized {passes} times" if passes > 1 else "")
                      + f" with the workload blocksize, absmax mode and output dtype "
                      f"(counter-based inputs; {c.description}), "
                      f"{threads} thread{'s' if threads > 1 else ''}, scalar C oracle"}


def cpu_baseline(cfg, target_s):
    """The oracle on all host threads (the reported baseline) and on one thread,
    each as the paper's protocol: one sizing / warm-up pass,
    then the mean of 3 measured passes of ~target/3 seconds."""
    def mean_of_3(threads, target):
        first = time_oracle(cfg, target_s=target / 3, threads=threads)      # sizes n, warms up
        n = first["elements"]
        runs = [time_oracle(cfg, threads=threads, n=n) for _ in range(3)]
        r = dict(runs[-1])
        r["value"] = round(statistics.mean(x["value"] for x in runs), 3)
        r["gelem_per_s"] = round(statistics.mean(x["gelem_per_s"] for x in runs), 4)
        r["seconds"] = round(sum(x["seconds"] for x in runs), 2)
        r["passes_gbs"] = [x["value"] for x in runs]
        r["sample"] += "; mean of 3 measured passes after a sizing / warm-up pass"
        return r
    multi = mean_of_3(len(os.sched_getaffinity(0)), target_s)
    one = mean_of_3(1, max(1.5, target_s / 2))
    multi["one_thread"] = {k: one[k] for k in ("value", "gelem_per_s", "seconds", "sample", "passes_gbs")}
    multi["threads_speedup"] = round(multi["gelem_per_s"] / max(one["gelem_per_s"], 1e-9), 2)
    return multi


def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg = args.config
    # each step is a bounded sample sized so the whole run takes ~90 s
    per_step = args.ref_step_seconds or max(0.2, min(5.0, 90.0 / max(1, args.steps + args.warmup)))
    threads = len(os.sched_getaffinity(0))
    n = size_oracle_sample(cfg, per_step, threads)
    first = time_oracle(cfg, threads=threads, n=n)          # re-size once from a full-size run
    n = int(min(1 << 31, max(1 << 22, n * per_step / max(first["seconds"], 1e-3))))
    n -= n % 16384
    steps = []
    for i in range(args.warmup + args.steps):
        cb = time_oracle(cfg, threads=threads, n=n)
        if i >= args.warmup:
            steps.append(cb)
    v = statistics.median(s["value"] for s in steps)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "u8->" + wl.CONFIGS[cfg].out_dtype, "data": "synthetic",
        "config": {"workload": wl.CONFIGS[cfg].description, "key": cfg},
        "ms_per_step": round(1000 * statistics.median(s["seconds"] for s in steps), 1),
        "cpu_baseline": {k: steps[-1][k] for k in ("kind", "cores", "sample")} | {"value": v, "unit": UNIT},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# work assignment and the cross-rank reduction (the only cross-rank traffic)
# ---------------------------------------------------------------------------
def rank_tensors(cfg: str, scaling: str, world: int, rank: int, layers=None, shard_of: int = 0):
    """Tensors rank `rank` dequantizes: its row shard of every weight (strong)
    or a full linear-weight set of its own (weak).  shard_of = S > 1 on one GPU:
    rank 0's shard of an S-way split (one GPU's work of an S-GPU run, e.g.
    config 4, whose full model does not fit one GPU)."""
    if shard_of > 1 and world == 1:
        return wl.config_tensors(cfg, world_size=shard_of, rank=0, layers=layers)
    if scaling == "strong":
        return wl.config_tensors(cfg, world_size=world, rank=rank, layers=layers)
    return wl.config_tensors(cfg, layers=layers)


def rank_seed0(cfg: str, rank: int) -> int:
    return 1000 * int(cfg[-1]) + 100000 * rank


def alg_bytes_of(tensors, blocksize: int, dq: bool) -> int:
    """SURVEY 8(d) algorithmic bytes of one pass over `tensors` (== WeightStore.algorithmic_bytes)."""
    tot = 0
    for t in tensors:
        nb = -(-t.n // blocksize)
        tot += (t.n + 1) // 2 + 2 * t.n + ((nb + 4 * (-(-nb // 256))) if dq else 4 * nb)
    return tot + (1024 if dq and tensors else 0)


def reduce_over_ranks(ms: float, alg_bytes: float, elems: float, device, world: int):
    """Max of the per-rank timed-region milliseconds and sum of the per-rank work
    (algorithmic bytes, elements) -- the only cross-rank traffic of the path."""
    import torch
    import torch.distributed as dist
    if world > 1 and dist.get_backend() == "gloo":
        device = "cpu"
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    u = torch.tensor([alg_bytes, elems], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(t.item()), float(u[0].item()), float(u[1].item())


def sum_over_ranks(x: float, device, world: int) -> float:
    import torch
    import torch.distributed as dist
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if dist.get_backend() == "gloo" else device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_per_rank(ms: float, device, world: int):
    import torch
    import torch.distributed as dist
    if world == 1:
        return [ms]
    if dist.get_backend() == "gloo":
        device = "cpu"
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [float(x.item()) for x in out]


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
L2_BYTES = 126e6


def replicas_for(alg_bytes: int) -> int:
    """Rotating copies of an L2-resident workload so that every timed step reads
    and writes data last touched > 4 x L2 bytes earlier (cold), 1 otherwise."""
    if alg_bytes > 8 * L2_BYTES:
        return 1
    return max(2, -(-int(4 * L2_BYTES) // max(1, alg_bytes)))


def build_store(args, cfg, rank, world, device):
    from synth import stores
    c = wl.CONFIGS[cfg]
    tensors = rank_tensors(cfg, args.scaling, world, rank, args.layers, args.shard_of)
    reps = replicas_for(alg_bytes_of(tensors, c.blocksize, c.dq))
    maker = stores.from_gaussian if args.inputs == "gaussian" else stores.from_hash
    return maker(tensors * reps, c.blocksize, c.dq, c.out_dtype, seed0=rank_seed0(cfg, rank), device=device), \
        tensors, reps


def measure_sol(nf4, torch, in_bytes=2 << 30, reps=10):
    src = torch.empty(in_bytes, dtype=torch.uint8, device="cuda")
    src.random_(0, 255)
    dst = torch.empty(4 * in_bytes, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        nf4.nf4_sol_stream(src, in_bytes, dst)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        nf4.nf4_sol_stream(src, in_bytes, dst)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    del src, dst
    torch.cuda.empty_cache()
    return round(5 * in_bytes / (ms * 1e-3) / 1e9, 1)


def pcie_link_rates(torch, nbytes=1 << 30):
    """Plain pinned-host <-> HBM copy rates (torch copy_, CUDA events, best of 3) --
    the ceiling of the e2e path, whose outputs must cross this link."""
    try:
        h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
        d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        s = torch.cuda.current_stream()
        res = {}
        for name, fn in (("d2h_gbs", lambda: h.copy_(d, non_blocking=True)),
                         ("h2d_gbs", lambda: d.copy_(h, non_blocking=True))):
            best = 1e30
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                fn()
                b.record(s)
                b.synchronize()
                best = min(best, a.elapsed_time(b))
            res[name] = round(nbytes / (best * 1e-3) / 1e9, 2)
        del h, d
        return res
    except Exception as e:   # pinned allocation refused: report nothing rather than fail the bench
        return {"error": str(e)[:120]}


def run_e2e(nf4, torch, ws, args, max_host_bytes, device=None, world=1):
    """Same metric through nf4_dequantize_host_batched: pinned host inputs -> HBM
    -> kernel -> pinned host outputs, copies inside the timed region."""
    bs = ws.blocksize
    # bounded prefix of the workload that fits the host-memory budget
    chosen, host_bytes = [], 0
    for i, e in enumerate(ws.entries):
        nb = -(-e.n // bs)
        b = (e.n + 1) // 2 + 2 * e.n + (nb + 4 * (-(-nb // 256)) if ws.dq else 4 * nb)
        if chosen and host_bytes + b > max_host_bytes:
            break
        chosen.append(i)
        host_bytes += b
    chunk = 1 << 24
    wsp = torch.empty(nf4.nf4_host_workspace_bytes(chunk, bs, ws.dq), dtype=torch.uint8, device="cuda")
    items, h2d, d2h, alg = [], 0, 0, 0
    code2_h = ws.code2.cpu().pin_memory() if ws.dq else None
    for i in chosen:
        e = ws.entries[i]
        nb = -(-e.n // bs)
        pk = ws.codes[e.codes_off:e.codes_off + (e.n + 1) // 2].cpu().pin_memory()
        out = torch.empty(e.n, dtype=torch.int16).pin_memory()
        if ws.dq:
            q = ws.scales[e.scale_off:e.scale_off + nb].cpu().pin_memory()
            a2 = ws.groups[e.group_off:e.group_off + 4 * (-(-nb // 256))].cpu().pin_memory()
            dq = nf4.DQ(q, code2_h, a2, e.offset)
            items.append((pk, None, dq, e.n, out))
            h2d += pk.numel() + q.numel() + a2.numel() + 1024
        else:
            a = ws.scales[e.scale_off:e.scale_off + 4 * nb].cpu().pin_memory()
            items.append((pk, a, None, e.n, out))
            h2d += pk.numel() + a.numel()
        d2h += 2 * e.n
        alg += (e.n + 1) // 2 + 2 * e.n + ((nb + 4 * (-(-nb // 256)) + 1024) if ws.dq else 4 * nb)

    descs = [nf4.NF4Tensor(pk, n, bs, out, a, dq) for pk, a, dq, n, out in items]

    def step():
        # one pipelined call over all tensors: pinned host -> HBM -> kernel -> pinned host
        nf4.nf4_dequantize_host_batched(descs, ws.out_dtype, workspace=wsp, chunk_elems=chunk)
        return nf4.nf4_last_launch_count()

    for _ in range(2):
        step()
    k = args.e2e_steps
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        step()                       # synchronous: returns with the outputs on the host
    dt = (time.perf_counter() - t0) / k
    del wsp
    # whole job: max time over ranks, summed work (the ranks stream concurrently)
    dt_ms, alg_all, elems_all = reduce_over_ranks(dt * 1e3, float(alg), float(sum(it[3] for it in items)),
                                                  device if device is not None else "cpu", world)
    dt = dt_ms * 1e-3
    link = pcie_link_rates(torch)
    if link and "d2h_gbs" in link:
        # the outputs (2 B per element, ~80% of the step's bytes) cross PCIe device->host
        link["e2e_d2h_gbs"] = round(d2h / (dt_ms * 1e-3) / 1e9, 2)
        link["e2e_d2h_frac_of_link"] = round(link["e2e_d2h_gbs"] / link["d2h_gbs"], 3)
    return {"value": round(alg_all / dt / 1e9, 2), "unit": UNIT, "h2d_bytes_per_step": int(h2d) * world,
            "pcie": link,
            "d2h_bytes_per_step": int(d2h) * world, "ms_per_step": round(dt * 1e3, 2),
            "gelem_per_s": round(elems_all / dt / 1e9, 3),
            "sample": f"first {len(chosen)} of {len(ws.entries)} tensors per rank "
                      f"({sum(it[3] for it in items) / 1e9:.2f} G elements) through nf4_dequantize_host_batched, "
                      f"pinned host buffers, {chunk}-element chunks"}


def ncu_traffic(cfg, inputs, variant, alg_per_launch):
    """DRAM bytes per launch of the dequant kernel from the committed ncu capture
    (profiles/ncu_traffic.json), scaled to this launch -- only if that capture was
    taken on exactly these kernel sources (source hash), variant and workload;
    otherwise None with the reason."""
    from paper_2604_02556_b200 import _build
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            tr = json.load(f)
    except Exception:
        return None, "no ncu capture committed"
    want = {"config": cfg, "inputs": inputs, "variant": variant, "source_hash": _build.source_hash(_build.DEQUANT_SOURCES)}
    stale = [k for k, v in want.items() if tr.get(k) != v]
    if stale:
        return None, "ncu capture does not match this run (" + ", ".join(stale) + ")"
    return int(tr["traffic_bytes_per_alg_byte"] * alg_per_launch), \
        f"ncu --set full capture {tr.get('source', '')}: DRAM bytes / algorithmic = {tr['traffic_bytes_per_alg_byte']:.5f}"


def measure_dequant(args, cfg, rank, world, device, nf4, torch, steps, full=True):
    """Build the workload, warm up, time `steps` steps (max over ranks).  Returns
    (result dict, store)."""
    import torch.distributed as dist
    from paper_2604_02556_b200 import _lib
    c = wl.CONFIGS[cfg]
    t_build = time.perf_counter()
    ws, tensors, reps = build_store(args, cfg, rank, world, device)
    torch.cuda.synchronize()
    # inputs are complete (synchronized) before any timed launch: early input reads are safe
    nf4.nf4_set_early_input_reads(bool(getattr(args, "early_inputs", False)))
    t_build = time.perf_counter() - t_build
    nt = len(tensors)
    alg_step = alg_bytes_of(tensors, c.blocksize, c.dq)        # one pass over the workload
    n_step = sum(t.n for t in tensors)

    descs = ws.nf4_tensors()
    rep_carrs = []                          # per replica: its launches (<= NF4_MAX_BATCH tensors each)
    for r in range(reps):
        d = descs[r * nt:(r + 1) * nt]
        groups = [d[i:i + _lib.NF4_MAX_BATCH] for i in range(0, len(d), _lib.NF4_MAX_BATCH)]
        rep_carrs.append([(_lib.TensorDesc * len(g))(*[x.c() for x in g]) for g in groups])
    carrs = rep_carrs[0]
    lib = nf4.load()
    odt = _lib.NF4_F16 if c.out_dtype == "f16" else _lib.NF4_BF16
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream or None
    launch_events = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in carrs]

    def step(timed_launches=None, i=0, s_ptr=None):
        n_launch = 0
        for gi, arr in enumerate(rep_carrs[i % reps]):
            if timed_launches is not None:
                timed_launches[gi][0].record(stream)
            st = lib.nf4_dequantize_batched(arr, len(arr), odt, s_ptr or sptr)
            if st != 0:
                raise _lib.NF4Error(st, "nf4_dequantize_batched")
            n_launch += lib.nf4_last_launch_count()
            if timed_launches is not None:
                timed_launches[gi][1].record(stream)
        return n_launch

    for i in range(max(args.warmup, reps)):
        step(i=i)
    torch.cuda.synchronize()

    # Small (L2-resident) workloads: `reps` rotating copies of the inputs and outputs
    # (> 4 x L2 in total), and the timed steps -- step i on copy i % reps -- are
    # launched back to back from ONE CUDA graph, so every step starts L2-cold and
    # the time per step is the graph's time / steps (no per-launch event or
    # host-launch floor).  The diagnostic per-launch pass below flushes L2 by
    # READING 512 MB between single launches instead.
    cold = reps > 1
    if cold:
        flush_buf = torch.ones(512 << 20, dtype=torch.uint8, device=device)
        flush_sink = torch.empty(1, dtype=torch.int64, device=device)

        def flush():
            flush_sink.copy_(flush_buf.sum(dtype=torch.int64))

    # diagnostic pass: CUDA events around every launch (breaks the PDL overlap
    # between launches, so it is slightly slower than the timed pass below)
    kt = []
    if full:
        for _ in range(max(3, min(steps, 20))):
            if cold:
                flush()
            step(launch_events)
            torch.cuda.synchronize()
            kt.append(sum(s.elapsed_time(e) for s, e in launch_events))

    sampler = ClockSampler(device.index if device.index is not None else 0) if full else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
        time.sleep(0.3)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = 0
    if cold:
        gs = torch.cuda.Stream(device=device)
        gs.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            for i in range(steps):
                launches += step(i=i, s_ptr=gs.cuda_stream)
        graph.replay()                       # warm-up replay (first replay uploads the graph)
        torch.cuda.synchronize()
        start.record(stream)
        graph.replay()
        end.record(stream)
    else:
        start.record(stream)
        for _ in range(steps):
            launches += step()
        end.record(stream)
    torch.cuda.synchronize()
    nf4.nf4_set_early_input_reads(False)   # back to the library default for anything after the timing
    if world > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    ms = start.elapsed_time(end)
    per_rank_ms = gather_per_rank(ms, device, world)
    ms_max, tot_bytes, tot_elems = reduce_over_ranks(ms, float(alg_step), float(n_step), device, world)
    launches_all = int(sum_over_ranks(float(launches), device, world))   # every rank's kernels
    value = tot_bytes * steps / (ms_max * 1e-3) / 1e9
    gelem = tot_elems * steps / (ms_max * 1e-3) / 1e9
    res = {"value": value, "gelem": gelem, "ms_max": ms_max, "ms_rank": ms, "per_rank_ms": per_rank_ms,
           "launches": launches, "launches_all": launches_all, "launches_per_step": len(carrs), "kt": kt, "clocks": clocks, "cold": cold,
           "reps": reps, "t_build": t_build, "tensors": tensors, "alg_per_step": alg_step, "n_rank": n_step,
           "tot_bytes": tot_bytes, "tot_elems": tot_elems}
    return res, ws


def f1_layer_groups(tensors):
    """Consecutive weights of one decoder layer that share X: (q,k,v), (o), (gate,up), (down)."""
    groups, cur = [], []
    for i, t in enumerate(tensors):
        kind = t.name.split(".")[2].split("[")[0]
        key = {"q_proj": "qkv", "k_proj": "qkv", "v_proj": "qkv", "gate_proj": "gu", "up_proj": "gu"}.get(kind, kind)
        lay = t.name.split(".")[1]
        if cur and (cur[0][1] != (lay, key) or key not in ("qkv", "gu")):
            groups.append([c[0] for c in cur])
            cur = []
        cur.append((i, (lay, key)))
    if cur:
        groups.append([c[0] for c in cur])
    return groups


# The fused GEMM's own bound: one shared-memory table lookup per weight costs 1/32 of a
# 128-B LSU data-pipe wavefront (16-entry table: LDS.32 per weight; byte-pair table:
# LDS.64 per two weights -- the same wavefronts), and that pipe sustains 6.48 T
# lookups/s on this GPU (tools/lutbench.cu, profiles/r01_lutbench.txt).
F1_LUT_BOUND = 6.48e12


def measure_f1(nf4, torch, peak, ms_list=(1, 16, 64), layers=8, steps=20, warmup=5):
    """Y_t = X_t . W_t^T for every linear weight of `layers`
    Gemma-3-27B decoder layers (DQ NF4, bf16 X/Y), fused vs the unfused path the
    paper optimizes (nf4_dequantize into a bf16 buffer, then cuBLAS via
    torch.matmul).  Fused, two ways: `fused_ms` keeps a decoder layer's data
    dependencies (q/k/v -> o -> gate/up -> down: one nf4_gemm_grouped launch for
    the weights sharing X, nf4_gemm otherwise, 4 launches per layer);
    `one_launch_ms` runs all the step's weights as independent problems in one
    nf4_gemm_multi launch (fill/drain paid once).
    HBM roofline of the fused step: the bytes it must move (codes + qabsmax +
    absmax2 + X + Y) over the measured copy peak."""
    from synth import stores
    tensors = wl.model_tensors("gemma-3-27b", layers=layers)
    ws = stores.from_hash(tensors, 64, True, "bf16", seed0=77, device="cuda")
    dqs = [nf4.DQ(ws._ptr(ws.scales, e.scale_off), ws.code2.data_ptr(), ws._ptr(ws.groups, e.group_off), e.offset)
           for e in ws.entries]
    groups = f1_layer_groups(tensors)
    n_total = sum(t.n for t in tensors)
    out = {"workload": f"Gemma-3-27B, {layers} decoder layers x 7 linear weights ({n_total / 1e9:.2f} G NF4 "
                       f"weights, blocksize 64, double-quant), bf16 X and Y",
           "launches_per_step": len(groups), "steps": steps,
           "roofline_note": "hbm_frac: bytes the fused step must move (codes + scales + X + Y) / time / measured "
                            "copy peak; lut_bound_frac: weights/s / 6.48 T lookups/s, the measured rate of the "
                            "shared-memory LSU data pipe for one table lookup per weight (the fused kernel's "
                            "binding pipe, ncu: l1tex ~80% busy in the one-launch step)"}
    wbuf = torch.empty(max(t.n for t in tensors), dtype=torch.bfloat16, device="cuda")
    for M in ms_list:
        xs = {}
        for t in tensors:
            if t.cols not in xs:
                xs[t.cols] = torch.randn(M, t.cols, device="cuda").to(torch.bfloat16)
        ys = [torch.empty(M, t.rows, dtype=torch.bfloat16, device="cuda") for t in tensors]
        gws = {}
        for g in groups:
            Ns = tuple(tensors[i].rows for i in g)
            K = tensors[g[0]].cols
            b = (nf4.nf4_gemm_grouped_workspace_bytes(M, Ns, K) if len(g) > 1
                 else nf4.nf4_gemm_workspace_bytes(M, Ns[0], K, 0))
            gws[tuple(g)] = torch.zeros(max(16, b), dtype=torch.uint8, device="cuda")

        def fused():
            for g in groups:
                K = tensors[g[0]].cols
                if len(g) == 1:
                    i = g[0]
                    nf4.nf4_gemm(xs[K], ws._ptr(ws.codes, ws.entries[i].codes_off), None, dqs[i], N=tensors[i].rows,
                                 K=K, y=ys[i], workspace=gws[tuple(g)])
                else:
                    members = [(ws._ptr(ws.codes, ws.entries[i].codes_off), None, dqs[i], tensors[i].rows) for i in g]
                    nf4.nf4_gemm_grouped(xs[K], members, K=K, ys=[ys[i] for i in g], workspace=gws[tuple(g)])

        mws = torch.zeros(max(16, nf4.nf4_gemm_multi_workspace_bytes(M, [t.rows for t in tensors],
                                                                     [t.cols for t in tensors])),
                          dtype=torch.uint8, device="cuda")
        probs = [(xs[t.cols], t.cols, ws._ptr(ws.codes, e.codes_off), None, dqs[i], t.rows)
                 for i, (t, e) in enumerate(zip(tensors, ws.entries))]

        def one_launch():
            # every weight of the step in ONE persistent launch (independent problems: the
            # decode-step inputs are all ready, e.g. batched / speculative / MoE-style use)
            nf4.nf4_gemm_multi(probs, M=M, ys=ys, workspace=mws)

        def unfused():
            for i, (t, e) in enumerate(zip(tensors, ws.entries)):
                nf4.nf4_dequantize(ws._ptr(ws.codes, e.codes_off), None, dqs[i], n=e.n, blocksize=64,
                                   out_dtype="bf16", out=wbuf)
                torch.matmul(xs[t.cols], wbuf[:e.n].view(t.rows, t.cols).t(), out=ys[i])

        def timeit(fn):
            for _ in range(warmup):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(steps):
                fn()
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b) / steps

        f_ms = timeit(fused)
        o_ms = timeit(one_launch) if len(probs) <= 64 else None
        u_ms = timeit(unfused)
        wbytes = sum(e.n // 2 + e.n // 64 + 4 * (e.n // 64 // 256) for e in ws.entries) + 1024
        xybytes = sum(2 * M * (t.cols + t.rows) for t in tensors)
        gbs = (wbytes + xybytes) / (f_ms * 1e-3) / 1e9
        out[f"M{M}"] = {"fused_ms": round(f_ms, 4), "unfused_ms": round(u_ms, 4),
                        "speedup_vs_dequant_plus_cublas": round(u_ms / f_ms, 3),
                        "weights_per_s_T": round(n_total / (f_ms * 1e-3) / 1e12, 3),
                        "tflops": round(2.0 * M * n_total / (f_ms * 1e-3) / 1e12, 2),
                        "hbm_gbs": round(gbs, 1), "hbm_frac": round(gbs / peak, 4),
                        "bytes_per_step": wbytes + xybytes}
        out[f"M{M}"]["lut_bound_frac"] = round(n_total / (f_ms * 1e-3) / F1_LUT_BOUND, 4)
        if o_ms is not None:
            gbs1 = (wbytes + xybytes) / (o_ms * 1e-3) / 1e9
            out[f"M{M}"]["one_launch_lut_bound_frac"] = round(n_total / (o_ms * 1e-3) / F1_LUT_BOUND, 4)
            out[f"M{M}"].update({"one_launch_ms": round(o_ms, 4),
                                 "one_launch_speedup_vs_dequant_plus_cublas": round(u_ms / o_ms, 3),
                                 "one_launch_weights_per_s_T": round(n_total / (o_ms * 1e-3) / 1e12, 3),
                                 "one_launch_hbm_frac": round(gbs1 / peak, 4)})
        del xs, ys, gws, mws, probs
    del ws, wbuf
    torch.cuda.empty_cache()
    return out


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2604_02556_b200 as nf4

    # NF4_BENCH_SHARED_GPU=1 (harness test only): every rank on cuda:0 with gloo, so the
    # whole N-rank path (launch, sharding, reductions, JSON line) runs on a 1-GPU box.
    # NCCL refuses two ranks on one device; the numbers of such a run are not a measurement.
    shared = os.environ.get("NF4_BENCH_SHARED_GPU") == "1"
    if not shared and torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: {world} ranks but only {torch.cuda.device_count()} visible GPUs")
    dev_index = 0 if shared else local_rank
    torch.cuda.set_device(dev_index)
    device = torch.device("cuda", dev_index)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=device)
    nf4.load()
    if args.variant is not None:
        nf4.nf4_set_kernel_variant(int(args.variant) if args.variant.isdigit() else args.variant)
    variant = nf4.nf4_kernel_variants()[nf4.nf4_get_kernel_variant()]
    c = wl.CONFIGS[args.config]
    peak, peak_src = _peaks()

    r, ws = measure_dequant(args, args.config, rank, world, device, nf4, torch, args.steps)
    alg_per_step = r["alg_per_step"]
    ms_per_step = r["ms_max"] / args.steps
    # roofline of the dominant (and only) kernel in the timed region: every launch there is
    # nf4::dequant_kernel, so its average launch duration is the timed region over the launches,
    # and the bytes of one launch are its share of the step's algorithmic bytes
    kernel_ms_per_launch = r["ms_rank"] / max(1, r["launches"])
    alg_per_launch = alg_per_step / r["launches_per_step"]
    achieved = alg_per_launch / (kernel_ms_per_launch * 1e-3) / 1e9
    traffic, traffic_note = ncu_traffic(args.config, args.inputs, variant, alg_per_launch)
    kt = r["kt"]

    extra = {}
    if rank == 0 and not args.no_sol:
        extra["sol_stream_gbs"] = measure_sol(nf4, torch)
    e2e = None
    if not args.no_e2e:
        try:
            import psutil
            avail = psutil.virtual_memory().available
        except Exception:
            avail = 16 << 30
        budget = int(min(avail // (4 * max(world, 1)), args.e2e_host_gb * (1 << 30)))
        e2e = run_e2e(nf4, torch, ws, args, budget, device=device, world=world)
    del ws
    torch.cuda.empty_cache()

    extra_cfgs = {}
    if world == 1 and args.extra_configs:
        for cfg in [x for x in args.extra_configs.split(",") if x and x != args.config]:
            rx, wsx = measure_dequant(args, cfg, rank, world, device, nf4, torch, max(10, args.steps // 2),
                                      full=False)
            del wsx
            torch.cuda.empty_cache()
            cx = wl.CONFIGS[cfg]
            extra_cfgs[cfg] = {"workload": cx.description, "value": round(rx["value"], 1), "unit": UNIT,
                               "gelem_per_s": round(rx["gelem"], 2),
                               "ms_per_step": round(rx["ms_max"] / max(10, args.steps // 2), 4),
                               "roofline_frac": round(rx["value"] / peak, 4),
                               "pct_of_nominal_8000": round(100 * rx["value"] / NOMINAL_HBM_GBS, 2),
                               "bytes_per_step": rx["alg_per_step"], "launches_per_step": rx["launches_per_step"],
                               "steps": max(10, args.steps // 2), "cold_l2": rx["cold"],
                               "rotating_copies": rx["reps"]}

    f1 = None
    if world == 1 and not args.no_f1:
        f1 = measure_f1(nf4, torch, peak)

    cb = None
    if rank == 0 and not args.no_cpu_baseline:
        cb = cpu_baseline(args.config, target_s=args.cpu_seconds)
    if world > 1:
        dist.barrier()

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(r["value"], 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None,
            "dtype": f"u8->{c.out_dtype}",
            "data": ("synthetic: W~N(0,0.02^2) per tensor (torch on device), quantized by nf4_quantize"
                     + (" + nf4_double_quantize" if c.dq else "")) if args.inputs == "gaussian"
                    else "synthetic: counter-based hash codes/scales (synth.inputs)",
            "config": {"workload": c.description, "key": args.config,
                       "model": c.model or "single 4096x4096", "tensors_per_rank": len(r["tensors"]),
                       "elements_per_rank": r["n_rank"], "elements_total": int(r["tot_elems"]),
                       "blocksize": c.blocksize, "absmax": "double-quant" if c.dq else "fp32",
                       "out_dtype": c.out_dtype, "algorithmic_bytes_per_step_per_rank": alg_per_step,
                       "algorithmic_bytes_per_step_total": int(r["tot_bytes"]),
                       "launches_per_step": r["launches_per_step"], "kernel_variant": variant,
                       "early_input_reads": bool(args.early_inputs),
                       "l2": "inputs+outputs per step >> 126 MB L2 (no flush needed)"
                             if not r["cold"] else f"L2-resident workload: {r['reps']} rotating copies "
                                                   f"(> 4 x L2), the {args.steps} timed steps launched back to back "
                                                   "from one CUDA graph (step i on copy i % copies); time = graph "
                                                   "replay / steps",
                       "shard_of": args.shard_of or None,
                       "parallelism": (f"row-sharded {world} ways (each rank its own shard of every weight), "
                                       "no data-path collective" if args.scaling == "strong"
                                       else f"{world} independent replicas") if world > 1 else "single GPU"},
            "gelem_per_s": round(r["gelem"], 2),
            "pct_of_peak": {"measured_copy_%.1f" % peak: round(100 * r["value"] / world / peak, 2),
                            "nominal_8000": round(100 * r["value"] / world / NOMINAL_HBM_GBS, 2)},
            "per_rank_ms_per_step": [round(x / args.steps, 4) for x in r["per_rank_ms"]],
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": UNIT,
                         "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_note,
                         "peak_source": peak_src, "kernel": "nf4::dequant_kernel",
                         "timing": "timed region of this run (rank 0) / its launches; every launch there is "
                                   "this kernel",
                         "kernel_ms_per_launch": round(kernel_ms_per_launch, 4),
                         "bytes_per_launch": int(alg_per_launch),
                         "pct_of_nominal_8000": round(100 * achieved / NOMINAL_HBM_GBS, 2),
                         # separate diagnostic pass with CUDA events around every launch (events between
                         # launches break the PDL overlap): median / best / worst and the paper's
                         # "mean of 3 measured passes after 1 warm-up"
                         "per_launch_events_gbs": None if not kt else {
                             "median": round(alg_per_step / (statistics.median(kt) * 1e-3) / 1e9, 1),
                             "best": round(alg_per_step / (min(kt) * 1e-3) / 1e9, 1),
                             "worst": round(alg_per_step / (max(kt) * 1e-3) / 1e9, 1),
                             "paper_mean_of_3": round(alg_per_step / (statistics.mean(kt[:3]) * 1e-3) / 1e9, 1),
                             "passes": len(kt)}},
            "e2e": e2e,
            "cpu_baseline": cb,
            "gpu_launches": r["launches_all"],
            "clocks": r["clocks"],
            "setup_seconds": round(r["t_build"], 1),
        }
        if extra_cfgs:
            line["extra_configs"] = extra_cfgs
        if f1 is not None:
            line["f1"] = f1
        line.update(extra)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_dry(args, rank, world):
    """--dry-run: the multi-rank harness without a GPU (gloo): work assignment,
    algorithmic bytes, the cross-rank reduction and the single JSON line, with a
    synthetic per-rank time.  Used by the CPU tests of the launch path."""
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    c = wl.CONFIGS[args.config]
    tensors = rank_tensors(args.config, args.scaling, world, rank, args.layers)
    alg = alg_bytes_of(tensors, c.blocksize, c.dq)
    ms = alg / 6.5e9 * args.steps * (1.0 + 0.01 * rank)
    per_rank = gather_per_rank(ms, "cpu", world)
    ms_max, tot_b, tot_e = reduce_over_ranks(ms, float(alg), float(sum(t.n for t in tensors)), "cpu", world)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": round(tot_b * args.steps / (ms_max * 1e-3) / 1e9, 1),
                          "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "scaling": args.scaling, "dry_run": True,
                          "config": {"key": args.config, "elements_total": int(tot_e),
                                     "algorithmic_bytes_per_step_total": int(tot_b),
                                     "tensors_per_rank": len(tensors)},
                          "per_rank_ms_per_step": [x / args.steps for x in per_rank]}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg3", choices=sorted(wl.CONFIGS))
    ap.add_argument("--layers", type=int, default=None, help="limit to the first L decoder layers")
    ap.add_argument("--inputs", default="gaussian", choices=["gaussian", "hash"])
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default=None, help="dequant kernel variant (name or index)")
    ap.add_argument("--extra-configs", default="cfg2,cfg1", help="comma list measured after the main config (N=1)")
    ap.add_argument("--early-inputs", action="store_true",
                    help="nf4_set_early_input_reads(1): inputs read before the PDL wait (include/nf4.h)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sol", action="store_true")
    ap.add_argument("--no-f1", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="no GPU: exercise the multi-rank harness with gloo")
    ap.add_argument("--shard-of", type=int, default=0,
                    help="N=1 only: time rank 0's row shard of an S-way split (config 4 per-GPU work)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-step-seconds", type=float, default=None,
                    help="oracle seconds per reference step (default: ~90 s / (steps + warmup), 0.2..5 s)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-host-gb", type=float, default=4.0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup raised to 3 (timing rule)", file=sys.stderr)
        args.warmup = 3
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        # not under torchrun: launch N local ranks of this same command
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] \
            + sys.argv[1:]
        sys.exit(subprocess.call(cmd, cwd=ROOT))
    rank = int(os.environ.get("RANK", "0"))
    world = int(env_world or "1")
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.dry_run:
        run_dry(args, rank, world)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
