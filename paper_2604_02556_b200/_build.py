"""Compile libnf4.so (the C-ABI library) in-tree for sm_100a with nvcc."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libnf4.so")
SOURCES = ["nf4_common.cu", "nf4_dequant.cu", "nf4_quantize.cu", "nf4_tools.cu", "nf4_gemm.cu"]
HEADERS = ["nf4_internal.cuh", os.path.join("..", "..", "include", "nf4.h"),
           os.path.join("..", "..", "include", "nf4_tools.h"), os.path.join("..", "..", "include", "nf4_gemm.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# No --use_fast_math, no -ftz=true: IEEE subnormals and RN division/multiply
# are part of the bit-exact contract.
NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC", "-shared",
              "-ftz=false", "-prec-div=true", "-prec-sqrt=true", "-fmad=false",
              "-cudart", "static", "-Xptxas", "-v"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, h) for h in HEADERS]
    return any(os.path.getmtime(d) > t for d in deps) or os.path.getmtime(__file__) > t


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *NVCC_FLAGS, "-o", tmp] + [os.path.join(CSRC, s) for s in SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libnf4.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, LIB)
    return LIB


def build_variant(name: str, defines: dict) -> str:
    """Diagnostics only (tools/): the same sources with extra -D macros, e.g.
    NF4_GEMM_DIAG=1 (event traces) or 2 (+ pipeline-skipping experiments), into
    <repo>/_variants/libnf4_<name>.so; load it with NF4_LIB=<path>."""
    out_dir = os.path.join(ROOT, "_variants")
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, f"libnf4_{name}.so")
    srcs = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, h) for h in HEADERS]
    if os.path.exists(out) and all(os.path.getmtime(d) <= os.path.getmtime(out) for d in srcs):
        return out
    cmd = [NVCC, *NVCC_FLAGS, *[f"-D{k}={v}" for k, v in defines.items()], "-o", out + ".tmp"] + \
        [os.path.join(CSRC, s) for s in SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building " + out)
    os.replace(out + ".tmp", out)
    return out


DEQUANT_SOURCES = ["nf4_common.cu", "nf4_dequant.cu", "nf4_internal.cuh", os.path.join("..", "..", "include", "nf4.h")]


def source_hash(files=None) -> str:
    """Hash of the sources a kernel is built from (default: everything in the
    library) plus the build flags: keys measurements such as
    profiles/ncu_traffic.json (the dequant kernel: DEQUANT_SOURCES) to the exact
    code they were taken on."""
    import hashlib
    h = hashlib.sha256()
    h.update(" ".join(NVCC_FLAGS).encode())
    for s in (files if files is not None else SOURCES + HEADERS):
        with open(os.path.join(CSRC, s), "rb") as f:
            h.update(s.encode() + b"\0" + f.read())
    return h.hexdigest()[:16]

if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
