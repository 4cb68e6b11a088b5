"""Fault injection into the parity checker ("failure
detection"): the comparisons every GPU parity test uses must fail when the
result is wrong, and pass when it is right.  The perturbation is injected in
the test harness, on a candidate result (the oracle's own output rounded to
fp32, i.e. what a correct fp32 kernel may return), never in the library:
the shipped code has no fault hooks.

* tolerance check (north_star: max |C - ref| / den <= 1e-5 for fp32):
  passes the rounded oracle output, fails a perturbation of 2e-5 * den in
  one element, and fails one NaN;
* bitwise check (integer-valued inputs, pin P4: every intermediate is exact,
  so any correct order gives the exact value): passes the exact result and
  fails a ONE-ULP flip of one element -- the smallest possible fault.
"""
import numpy as np

import datagen
import oracle

TOL32 = 1e-5


def _case(M=13, N=11, K=17, batch=9, seed=5, integers=False):
    ids = np.arange(batch, dtype=np.int64)
    A = datagen.fill_host(seed, datagen.MAT_A, np.float32, M, K, M, M * K, ids)
    B = datagen.fill_host(seed, datagen.MAT_B, np.float32, K, N, K, K * N, ids)
    C = datagen.fill_host(seed, datagen.MAT_C, np.float32, M, N, M, M * N, ids)
    if integers:  # entries in {-8..8}: exact in fp32 in any summation order (P4)
        A, B, C = (np.round(x * 8).astype(np.float32) for x in (A, B, C))
    ref, den, _ = oracle.ref_gemm("N", "N", M, N, K, 1.5, A, M, M * K, B, K, K * N, 0.5, C, M, M * N, batch)
    return ref, den


def test_tolerance_check_passes_a_correct_fp32_result():
    ref, den = _case()
    got = ref.astype(np.float32).astype(np.float64)  # a correctly rounded fp32 answer
    assert oracle.max_rel_err(got, ref, den) <= TOL32


def test_tolerance_check_catches_an_injected_error():
    ref, den = _case()
    got = ref.astype(np.float32).astype(np.float64)
    rng = np.random.default_rng(0)
    b, j, i = (int(rng.integers(0, s)) for s in got.shape)
    bad = got.copy()
    bad[b, j, i] += 2e-5 * den[b, j, i]  # twice the tolerance, one element of one problem
    assert oracle.max_rel_err(bad, ref, den) > TOL32
    nan = got.copy()
    nan[b, j, i] = np.nan
    assert oracle.max_rel_err(nan, ref, den) == np.inf


def test_bitwise_check_catches_a_one_ulp_flip():
    ref, den = _case(integers=True)
    exact = ref.astype(np.float32)
    assert np.array_equal(exact.astype(np.float64), ref)  # P4: the fp32 result is the exact one
    rng = np.random.default_rng(1)
    for _ in range(16):
        b, j, i = (int(rng.integers(0, s)) for s in exact.shape)
        bad = exact.copy()
        bad[b, j, i] = np.nextafter(bad[b, j, i], np.float32(np.inf))  # one ulp
        assert not np.array_equal(bad.view(np.int32), exact.view(np.int32))
        assert oracle.max_rel_err(bad.astype(np.float64), ref, den) > 0
