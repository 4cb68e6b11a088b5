"""Host code under AddressSanitizer + UndefinedBehaviorSanitizer (SURVEY
section 5): the run-time planner (csrc/planner.cpp, via tools/asan_planner.cpp
over a grid of inputs incl. domain edges, padding, misalignment, pointer
arrays, every dtype and transposition, plus the paper-faithful tiler) and the
C oracle (oracle/ref_gemm.c, via tools/asan_oracle.c with exact-fit
buffers).  compute-sanitizer is closed on the GPU pool, so device
memory safety is covered by the canary / padding / gap tests of the GPU suite."""
import os
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = ["-O1", "-g", "-fsanitize=address,undefined", "-fno-omit-frame-pointer", "-fno-sanitize-recover=all"]


def _build(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
    if r.returncode != 0 and "sanitize" in r.stderr and "unrecognized" in r.stderr:
        pytest.skip("compiler without sanitizers")
    assert r.returncode == 0, r.stderr[-3000:]


def _run(exe):
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=0:abort_on_error=1", UBSAN_OPTIONS="halt_on_error=1")
    r = subprocess.run([exe], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0 and "ERROR" not in r.stderr and "runtime error" not in r.stderr, \
        r.stdout[-1000:] + r.stderr[-4000:]
    return r.stdout


def test_planner_under_asan_ubsan():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "asan_planner")
        _build(["g++", "-std=c++17"] + SAN + ["-I", "paper_2208_09822_b200/csrc", "-I", "include", "-o", exe,
                                              "tools/asan_planner.cpp", "paper_2208_09822_b200/csrc/planner.cpp",
                                              "-ldl"])
        out = _run(exe)
    assert "planned" in out


def test_oracle_under_asan_ubsan():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "asan_oracle")
        _build(["gcc"] + SAN + ["-fopenmp", "-o", exe, "tools/asan_oracle.c", "oracle/ref_gemm.c", "-lm"])
        out = _run(exe)
    assert "oracle calls" in out
