"""CPU-side checks of the C ABI: the library loads without a GPU, exports
every symbol include/iaat.h declares, and the host-only entry points
(predicate, planner description, catalog) behave."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "iaat.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(iaat_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2208_09822_b200 import iaat
    declared = header_functions()
    assert set(declared) == set(iaat.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", iaat.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(iaat_\w+)", out))
    missing = set(declared) - exported
    assert not missing, missing
    lib = ctypes.CDLL(iaat.LIB_PATH)
    for name in declared:
        assert getattr(lib, name)


def test_small_predicate_matches_paper_examples():
    import json
    from paper_2208_09822_b200 import iaat
    cases = json.load(open(os.path.join(ROOT, "tests", "golden", "predicate.json")))["cases"]
    for c in cases:
        assert iaat.iaat_is_small_gemm(c["transA"], c["transB"], c["M"], c["N"], c["K"]) == c["small"], c
    assert not iaat.iaat_is_small_gemm("C", "N", 2, 2, 2)
    assert not iaat.iaat_is_small_gemm("N", "N", -1, 2, 2)


def test_tn_limit_extension():
    """the TN bound (paper: 32^3) can be widened up to 80^3 and
    restored; out-of-range requests are rejected and change nothing."""
    from paper_2208_09822_b200 import iaat
    assert iaat.iaat_get_tn_limit() == 32768
    assert not iaat.iaat_is_small_gemm("T", "N", 33, 32, 32)
    assert iaat.iaat_set_tn_limit(32767) == 1 and iaat.iaat_set_tn_limit(512001) == 1
    assert iaat.iaat_get_tn_limit() == 32768
    try:
        assert iaat.iaat_set_tn_limit(512000) == 0
        assert iaat.iaat_is_small_gemm("T", "N", 80, 80, 80)
        assert not iaat.iaat_is_small_gemm("T", "N", 81, 80, 80)
        assert iaat.iaat_is_small_gemm("N", "T", 80, 80, 80)  # other transpositions unchanged
        assert iaat.iaat_set_tn_limit(64000) == 0
        assert iaat.iaat_is_small_gemm("T", "N", 40, 40, 40) and not iaat.iaat_is_small_gemm("T", "N", 41, 40, 40)
        p = iaat.iaat_plan_describe(0, "T", "N", 40, 40, 40, 40, 1600, 40, 1600, 40, 1600, 1000)
        assert p.get("family")
    finally:
        assert iaat.iaat_set_tn_limit(32768) == 0
    assert not iaat.iaat_is_small_gemm("T", "N", 40, 40, 40)


def test_status_strings_and_version():
    from paper_2208_09822_b200 import iaat
    for k, v in iaat.STATUS.items():
        assert iaat.iaat_status_string(k) == v
    assert iaat.iaat_version() >= 100


def test_no_gpu_call_fails_cleanly():
    """Without a GPU a valid call returns a status (never crashes, never
    computes on the CPU)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2208_09822_b200 import iaat
    st = iaat.iaat_gemm_strided_batched(0, "N", "N", 4, 4, 4, 1.0, 256, 4, 16, 512, 4, 16, 0.0, 1024, 4, 16, 2)
    assert st in (3, 4)
    assert iaat.iaat_status_string(st).startswith("IAAT_ERROR")


def test_grouped_validation_before_any_launch():
    """every group is validated before anything is enqueued; the
    errors come back as statuses with no device involved (no GPU here)."""
    from paper_2208_09822_b200 import iaat
    g = dict(transA="N", transB="N", M=4, N=4, K=4, alpha=1.0, A=256, lda=4, strideA=16, B=512, ldb=4, strideB=16,
             beta=0.0, C=1024, ldc=4, strideC=16, batch=2)
    assert iaat.iaat_gemm_grouped_strided(0, []) == 0
    assert iaat.iaat_gemm_grouped_strided(0, [g, dict(g, lda=2)]) == 1          # INVALID_VALUE (lda < M)
    assert iaat.iaat_gemm_grouped_strided(0, [g, dict(g, transA="C")]) == 1      # INVALID_VALUE (op)
    assert iaat.iaat_gemm_grouped_strided(0, [dict(g, M=81, N=81, K=81, lda=81, ldb=81, ldc=81,
                                                    strideC=6561)]) == 2          # NOT_SMALL
    assert iaat.iaat_gemm_grouped_strided(0, [dict(g, strideC=3)]) == 1          # overlapping C
    assert iaat.iaat_gemm_grouped_strided(2, [dict(g, alpha=1j, beta=0.5 - 1j), dict(g, lda=1)]) == 1
