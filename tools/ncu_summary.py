#!/usr/bin/env python
"""Summarize ncu outputs for profiles/.

    python tools/ncu_summary.py --launches gpurun_out/launches_r01.csv \
        --rep gpurun_out/prof_dequant_r01.ncu-rep --alg-bytes-per-elem 2.515869 \
        --out profiles/r02_ncu_summary.md --traffic-json profiles/ncu_traffic.json --config cfg3

* launch list (`--metrics gpu__time_duration.sum,dram__bytes_*`): per-kernel
  time share and per-launch DRAM bytes vs the algorithmic bytes of the launch
  (written bytes / 2 = elements of a dequant launch);
* full capture: the raw metrics the roofline needs (DRAM bytes, duration,
  throughput %, stall reasons, registers, occupancy).
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess


def parse_launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        per.setdefault(r[ii], {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    return per


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return [dict(zip(r[0], row)) for row in r[2:]], dict(zip(r[0], r[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--alg-bytes-per-elem", type=float, default=2.515869140625)
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic-json")
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--variant", default="v2u4sxc", help="dequant kernel variant the capture ran")
    ap.add_argument("--title", default="ncu summary")
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    ratios = []
    if a.launches:
        per = parse_launches(a.launches)
        tot = collections.defaultdict(float)
        cnt = collections.Counter()
        for v in per.values():
            k = v["name"].split("(")[0]
            tot[k] += v.get("gpu__time_duration.sum", 0.0)
            cnt[k] += 1
        all_t = sum(tot.values())
        lines += [f"Launch list: `{a.launches}` ({len(per)} launches, cold-cache and serialised under ncu).", "",
                  "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for k, t in sorted(tot.items(), key=lambda x: -x[1]):
            lines.append(f"| `{k[:90]}` | {cnt[k]} | {t / 1e6:.3f} | {100 * t / all_t:.1f}% |")
        deq = [v for v in per.values() if "dequant_kernel" in v["name"]]
        if deq:
            step_share = sum(v["gpu__time_duration.sum"] for v in deq)
            lines += ["", f"Dequant launches: {len(deq)}; they are {100 * step_share / all_t:.1f}% of all GPU time "
                          "in this command (the rest is input generation: randn, nf4_quantize, mean, "
                          "nf4_double_quantize, which run once before the timed region).", "",
                      "| launch | us | DRAM read GB | DRAM write GB | elements (write/2) | algorithmic GB | traffic / algorithmic | DRAM GB/s |",
                      "|---|---|---|---|---|---|---|---|"]
            for i, v in enumerate(deq):
                rd, wr, t = v["dram__bytes_read.sum"], v["dram__bytes_write.sum"], v["gpu__time_duration.sum"]
                n = wr / 2
                alg = n * a.alg_bytes_per_elem
                ratios.append((rd + wr) / alg)
                lines.append(f"| {i} | {t / 1e3:.1f} | {rd / 1e9:.3f} | {wr / 1e9:.3f} | {n / 1e9:.3f} G | "
                             f"{alg / 1e9:.3f} | {(rd + wr) / alg:.4f} | {(rd + wr) / t:.0f} |")
    if a.rep:
        ms, units = raw_metrics(a.rep)
        keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
                "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
                "smsp__inst_executed.sum", "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
                "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
                "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
                "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
        lines += ["", f"Full capture: `{a.rep}`", "", "| metric | value | unit |", "|---|---|---|"]
        for m in ms:
            for k in keys:
                if k in m:
                    lines.append(f"| {k} | {m[k]} | {units.get(k, '')} |")
            try:
                rd = float(m["dram__bytes_read.sum"].replace(",", ""))
                wr = float(m["dram__bytes_write.sum"].replace(",", ""))
                ru, wu = units.get("dram__bytes_read.sum", ""), units.get("dram__bytes_write.sum", "")
                mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                rd *= mult.get(ru, 1)
                wr *= mult.get(wu, 1)
                n = wr / 2
                alg = n * a.alg_bytes_per_elem
                lines.append(f"| traffic / algorithmic bytes | {(rd + wr) / alg:.4f} | (elements = write bytes / 2) |")
                ratios.append((rd + wr) / alg)
            except (KeyError, ValueError):
                pass
            lines.append("| | | |")
    with open(a.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if a.traffic_json and ratios:
        with open(a.traffic_json, "w") as f:
            import os
            import sys
            sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
            from paper_2604_02556_b200 import _build
            # keyed to the kernel sources, variant and workload it was taken on: bench.py
            # reports roofline.traffic only while all of these still match
            json.dump({"config": a.config, "inputs": "gaussian", "variant": a.variant,
                       "source_hash": _build.source_hash(_build.DEQUANT_SOURCES),
                       "traffic_bytes_per_alg_byte": sum(ratios) / len(ratios),
                       "source": [a.launches, a.rep], "n_launches": len(ratios)}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
