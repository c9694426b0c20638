#!/usr/bin/env python
"""CPU oracle throughput per BASELINE configuration on this host: 1 thread and all
threads, ~target seconds each (the oracle as it stands; bench.py's sampling).
Prints one JSON line per configuration."""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    target = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
    for cfg in ("cfg1", "cfg2", "cfg3", "cfg4"):
        multi = bench.time_oracle(cfg, target_s=target)
        one = bench.time_oracle(cfg, target_s=target, threads=1)
        print(json.dumps({"config": cfg, "threads": multi["cores"], "gelem_per_s_T": multi["gelem_per_s"],
                          "gbs_T": multi["value"], "gelem_per_s_1": one["gelem_per_s"], "gbs_1": one["value"]}),
              flush=True)


if __name__ == "__main__":
    main()
