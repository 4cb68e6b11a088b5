"""Build checks on the sm_100a objects (CPU only, no GPU): register spills
within each family's budget in every generated kernel and none in any kernel
the bench configs use (ptxas reports kept by build.py), and the
SASS of the shipped library contains the instructions the design claims:
UBLKCP (cp.async.bulk HBM->SMEM staging), SYNCS (mbarrier), DMMA (fp64
tensor cores), FFMA, and no HMMA/tensor-op on the fp32 path (IEEE fp32)."""
import functools
import glob
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "build", "iaat")
LIB = os.path.join(ROOT, "paper_2208_09822_b200", "libiaat.so")


def _spill_reports():
    """(log, kernel, spill store bytes, spill load bytes) for every kernel of
    every translation unit build.py compiled (ptxas -v reports)."""
    out = []
    for lg in sorted(glob.glob(os.path.join(BUILD, "ptxas_*.log"))):
        txt = open(lg).read()
        for m in re.finditer(r"Compiling entry function '(\w+)'.*?(\d+) bytes spill stores, (\d+) bytes spill loads",
                             txt, re.S):
            out.append((os.path.basename(lg), m.group(1), int(m.group(2)), int(m.group(3))))
    return out


# Spill budgets per kernel family (bytes of spill stores).  The slab kernels
# (k_*), the fp64 / ZGEMM DMMA kernels (ksd_, ksz_) and the ksg kernels are
# spill-free; the K-streamed FMA kernels (ks1_, ksu_, ks_) may keep up to
# 16 words outside the k loop (install-time budget, gen/generate.py
# SPILL_EXCLUDE drops entries above it).
BUDGET = {"ptxas_api": 0, "ptxas_k_": 0, "ptxas_ksd_": 0, "ptxas_ksz_": 0, "ptxas_ksg_": 0, "ptxas_ksgs_": 0,
          "ptxas_ks1_": 64, "ptxas_ksu_": 64, "ptxas_ks_": 64}


def test_no_spills_in_any_kernel():
    reps = _spill_reports()
    if not reps:
        pytest.skip("no ptxas logs (library built elsewhere)")
    fams = set()
    for lg, kern, st, ld in reps:
        fam = next((f for f in sorted(BUDGET, key=len, reverse=True) if lg.startswith(f)), None)
        assert fam is not None, "no spill budget for %s" % lg
        fams.add(fam)
        assert st <= BUDGET[fam] and ld <= 4 * BUDGET[fam], (lg, kern, st, ld)
    assert {"ptxas_k_", "ptxas_ksd_", "ptxas_ksz_", "ptxas_ksg_", "ptxas_ks1_"} <= fams, fams


def test_kernels_used_by_the_bench_configs_do_not_spill():
    """Every kernel a plan of configs 1-7 selects (tuning table or cost model,
    host-only planning) has a spill-free ptxas report."""
    if not _spill_reports():
        pytest.skip("no ptxas logs (library built elsewhere)")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "used_kernels.py")], capture_output=True,
                       text=True, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " 0 spill" in r.stdout


@functools.lru_cache(maxsize=1)
def _sass():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout


def test_sass_has_bulk_copies_mbarriers_dmma():
    sass = _sass()
    assert "UBLKCP" in sass, "cp.async.bulk staging missing"
    assert "UTMALDG" in sass, "TMA tensor-map staging (K-streamed family) missing"
    assert "SYNCS" in sass, "mbarrier ops missing"
    assert "DMMA" in sass, "fp64 DMMA tensor-core path missing"
    assert "FFMA" in sass and "DFMA" in sass
    assert "arch = sm_100a" in sass or "sm_100a" in sass


def test_fp32_kernels_use_no_tensor_cores():
    sass = _sass()
    # split per function; fp32 kernels must not contain HMMA (TF32/F16 MMAs)
    funcs = re.split(r"\n\s*Function : ", sass)
    f32 = [f for f in funcs if "_f32" in f.split("\n", 1)[0] and "iaat" in f.split("\n", 1)[0]]
    assert f32
    for f in f32:
        assert "HMMA" not in f and "UTCHMMA" not in f and "DMMA" not in f
