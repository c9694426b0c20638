"""CPU-only checks of the C-ABI boundary: the library builds for sm_100a, loads
without a GPU, exports every symbol the headers declare, and validates
arguments (status codes) before touching the device."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2604_02556_b200 import _build, _lib
    _build.build()
    return _lib.load()


def _declared_symbols():
    names = set()
    for h in ("nf4.h", "nf4_tools.h", "nf4_gemm.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(nf4_[a-z0-9_]+)\s*\(", src):
            names.add(m.group(1))
    return names


def test_headers_declare_binding_exports():
    from paper_2604_02556_b200 import _lib
    assert _declared_symbols() == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    from paper_2604_02556_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    missing = _declared_symbols() - exported
    assert not missing, missing
    for name in _declared_symbols():
        assert hasattr(lib, name)


def test_library_is_sm100a_with_256bit_stores(lib):
    from paper_2604_02556_b200 import _lib
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH],
                          capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", _lib.LIB_PATH],
                                       capture_output=True, text=True).stdout
    assert "dequant_kernel" in sass
    assert "STG.E.EF.ENL2.256" in sass          # 256-bit evict-first output stores
    assert "LDG.E.NA.64.CONSTANT" in sass       # non-allocating read-only code loads
    assert "FFMA" not in _kernel_sass(sass, "dequant_kernel")  # product never contracted
    g = _kernel_sass(sass, "nf4_gemm_kernel")                   # F1: tcgen05 MMA + TMEM loads
    assert "UTCHMMA" in g and "LDTM" in g and "FFMA" not in g


def _kernel_sass(sass, name):
    parts = sass.split("Function : ")
    return "\n".join(p for p in parts if p.split("\n", 1)[0].find(name) >= 0)


def test_codebook_matches_table(lib):
    import paper_2604_02556_b200 as nf4
    cb = np.array(nf4.nf4_codebook(), np.float32)
    assert cb.view(np.uint32).tolist()[0] == 0xBF800000 and cb[7] == 0 and cb[15] == 1.0
    assert np.all(np.diff(cb) > 0)


def test_status_strings(lib):
    import paper_2604_02556_b200 as nf4
    for s in range(8):
        assert nf4.status_string(s).startswith("NF4_")


def test_argument_validation_without_gpu(lib):
    """Validation happens before any CUDA call, so it runs on the CPU host."""
    P = ctypes.c_void_p
    fake = P(0x1000)  # never dereferenced: every call below must fail validation first
    # negative n
    assert lib.nf4_dequantize(fake, fake, None, -1, 64, 0, fake, None) == 2
    # bad blocksize
    for bs in (0, 32, 96, 8192):
        assert lib.nf4_dequantize(fake, fake, None, 128, bs, 0, fake, None) == 3
    # bad dtype
    assert lib.nf4_dequantize(fake, fake, None, 128, 64, 2, fake, None) == 4
    # neither absmax nor dq
    assert lib.nf4_dequantize(fake, None, None, 128, 64, 0, fake, None) == 6
    # null pointers
    assert lib.nf4_dequantize(None, fake, None, 128, 64, 0, fake, None) == 1
    assert lib.nf4_dequantize(fake, fake, None, 128, 64, 0, None, None) == 1
    # misaligned fp32 absmax / 16-bit output
    assert lib.nf4_dequantize(fake, P(0x1001), None, 128, 64, 0, fake, None) == 5
    assert lib.nf4_dequantize(fake, fake, None, 128, 64, 0, P(0x1001), None) == 5
    # n == 0 is a no-op
    assert lib.nf4_dequantize(None, fake, None, 0, 64, 0, None, None) == 0
    # DQ state: blocksize2 must be 256
    from paper_2604_02556_b200._lib import DQState
    bad = DQState(fake, fake, fake, 0.0, 128)
    assert lib.nf4_dequantize(fake, None, ctypes.byref(bad), 128, 64, 0, fake, None) == 6
    # quantize / double quantize
    assert lib.nf4_quantize(fake, 7, 128, 64, fake, fake, None) == 4
    assert lib.nf4_quantize(fake, 2, 128, 48, fake, fake, None) == 3
    assert lib.nf4_double_quantize(fake, 10, 0.0, fake, 64, fake, fake, None) == 6
    # host path: chunk must be a multiple of 256*blocksize
    assert lib.nf4_dequantize_host(fake, fake, None, 1 << 20, 64, 0, fake, P(0x10000), 1 << 30, 1000, None) == 2
    # batched: negative count
    assert lib.nf4_dequantize_batched(None, -1, 0, None) == 2
    # fused GEMM: K not a multiple of 64, bad dtypes, misaligned X, both / neither scale modes
    assert lib.nf4_gemm(fake, 1, 4, fake, fake, None, 128, 100, 64, fake, 1, 0, None, 0, None) == 2
    assert lib.nf4_gemm(fake, 2, 4, fake, fake, None, 128, 128, 64, fake, 1, 0, None, 0, None) == 4
    assert lib.nf4_gemm(fake, 1, 4, fake, fake, None, 128, 128, 64, fake, 7, 0, None, 0, None) == 4
    assert lib.nf4_gemm(P(0x1008), 1, 4, fake, fake, None, 128, 128, 64, fake, 1, 0, None, 0, None) == 5
    assert lib.nf4_gemm(fake, 1, 4, fake, None, None, 128, 128, 64, fake, 1, 0, None, 0, None) == 6
    assert lib.nf4_gemm(fake, 1, 4, fake, fake, None, 128, 128, 48, fake, 1, 0, None, 0, None) == 3
    assert lib.nf4_gemm(fake, 1, 0, fake, fake, None, 128, 128, 64, fake, 1, 0, None, 0, None) == 0   # M == 0
    # grouped GEMM: count outside [1, 4], NULL table, a member with neither scale mode
    from paper_2604_02556_b200._lib import GemmWeight
    ws = (GemmWeight * 5)()
    for w in ws:
        w.packed, w.absmax, w.N, w.y = fake, fake, 128, fake
    assert lib.nf4_gemm_grouped(fake, 1, 4, 128, 64, ws, 0, 1, None, 0, None) == 2
    assert lib.nf4_gemm_grouped(fake, 1, 4, 128, 64, ws, 5, 1, None, 0, None) == 2
    assert lib.nf4_gemm_grouped(fake, 1, 4, 128, 64, None, 2, 1, None, 0, None) == 1
    ws[1].absmax = None
    assert lib.nf4_gemm_grouped(fake, 1, 4, 128, 64, ws, 2, 1, None, 0, None) == 6   # dq state unset (blocksize2 0)
    ws[1].dq.blocksize2 = 256
    assert lib.nf4_gemm_grouped(fake, 1, 4, 128, 64, ws, 2, 1, None, 0, None) == 1   # dq with NULL pointers
    assert lib.nf4_gemm_grouped_workspace_bytes(4, None, 2, 128) == 0


def test_binding_raises_loudly_without_library(tmp_path, monkeypatch):
    from paper_2604_02556_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        _lib.load()


def test_product_never_imports_oracle():
    """The product package shares no code with oracle/ (DESIGN.md 'Oracle')."""
    pkg = os.path.join(ROOT, "paper_2604_02556_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "oracle.h" not in src and "liboracle" not in src, f


def test_product_never_imports_test_inputs():
    """The product package does not import synth/ (the test-input generators)."""
    pkg = os.path.join(ROOT, "paper_2604_02556_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import synth" not in src and "from synth" not in src, f


def test_package_code2_table_equals_test_input_table():
    import numpy as np
    from paper_2604_02556_b200.tables import bnb_dynamic_code2
    from synth import inputs as syn
    a, b = bnb_dynamic_code2(), syn.dynamic_map_code2()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert a[127] == 0.0 and a[255] == 1.0 and np.all(np.diff(a) > 0)


def test_gemm_multi_validation_without_gpu(lib):
    """nf4_gemm_multi validates every problem before any CUDA call."""
    P = ctypes.c_void_p
    fake = P(0x1000)
    from paper_2604_02556_b200._lib import GemmProblem
    pr = (GemmProblem * 65)()
    for q in pr:
        q.x, q.K, q.packed, q.absmax, q.N, q.y = fake, 256, fake, fake, 128, fake
    assert lib.nf4_gemm_multi(pr, 0, 4, 1, 64, 1, None, 0, None) == 2       # count < 1
    assert lib.nf4_gemm_multi(pr, 65, 4, 1, 64, 1, None, 0, None) == 2      # count > NF4_GEMM_MAX_MULTI
    assert lib.nf4_gemm_multi(None, 2, 4, 1, 64, 1, None, 0, None) == 1     # NULL table
    assert lib.nf4_gemm_multi(pr, 2, 4, 2, 64, 1, None, 0, None) == 4       # x dtype fp32
    pr[1].K = 96                                                             # K not a multiple of 64
    assert lib.nf4_gemm_multi(pr, 2, 4, 1, 64, 1, None, 0, None) == 2
    pr[1].K = 128
    assert lib.nf4_gemm_multi(pr, 2, 4, 1, 256, 1, None, 0, None) == 2      # K not a multiple of blocksize
    pr[1].x = P(0x1008)                                                      # X not 16-byte aligned
    assert lib.nf4_gemm_multi(pr, 2, 4, 1, 64, 1, None, 0, None) == 5
    pr[1].x = None
    assert lib.nf4_gemm_multi(pr, 2, 4, 1, 64, 1, None, 0, None) == 1
    pr[1].x = fake
    pr[1].K = 0                                                              # K == 0: Y = 0, y still required
    pr[1].y = None
    assert lib.nf4_gemm_multi(pr, 2, 4, 1, 64, 1, None, 0, None) == 1
    # workspace sizing skips problems without work, as the call does
    N = (ctypes.c_int32 * 3)(128, 0, 256)
    K = (ctypes.c_int32 * 3)(512, 512, 0)
    N1 = (ctypes.c_int32 * 1)(128)
    K1 = (ctypes.c_int32 * 1)(512)
    assert lib.nf4_gemm_multi_workspace_bytes(4, N, K, 3) == lib.nf4_gemm_multi_workspace_bytes(4, N1, K1, 1)
    K[0] = 100
    assert lib.nf4_gemm_multi_workspace_bytes(4, N, K, 3) == 0
