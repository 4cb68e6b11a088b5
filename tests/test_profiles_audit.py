"""P12 -- FLOP and DRAM audit of committed ncu counters (profiles/audit_r01.json,
written by tools/audit.py from one ncu launch per case on a B200).

Exact tiles mean no padded or predicated work: FMA thread-instructions
(FFMA + 2 FFMA2, or 256 DMMA.8x8x4 + DFMA) equal M*N*K*batch plus the
epilogue's one FMA per C element when beta != 0, exactly.  No pack pass and
no re-reads: DRAM bytes read equal the algorithmic input bytes
(M*K + K*N + [beta != 0]*M*N) * elt * batch within 1 %."""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
AUDIT = os.path.join(ROOT, "profiles", "audit_r01.json")


def test_audit_covers_both_families_and_dtypes():
    d = json.load(open(AUDIT))
    kernels = " ".join(v["kernel"] for v in d.values())
    assert "iaat_f32_" in kernels and "iaat_ksu_f32_" in kernels and "iaat_ksd_f64_" in kernels
    assert len(d) >= 8


def test_fma_count_is_exact():
    for name, v in json.load(open(AUDIT)).items():
        m = re.match(r"(f32|f64)_(..)_(\d+)x(\d+)x(\d+)_b(\d+)_beta([0-9.]+)", name)
        M, N, K, batch, beta = int(m[3]), int(m[4]), int(m[5]), int(m[6]), float(m[7])
        want = M * N * K * batch + (M * N * batch if beta != 0 else 0)
        assert v["expected"] == want, name
        assert v["fma_thread_inst"] == want, (name, v["fma_thread_inst"], want)


def test_dram_reads_are_the_algorithmic_bytes():
    for name, v in json.load(open(AUDIT)).items():
        assert 1.0 <= v["read_ratio"] < 1.01, (name, v["read_ratio"])
