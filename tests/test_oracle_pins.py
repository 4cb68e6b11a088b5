"""Pins for the CPU oracle (oracle/ref_gemm.c) -- CPU only (-m "not gpu").

Each test checks the oracle against something other than itself: values the
paper / SPEC print, closed forms, invariants, exact rational arithmetic on
dense matrices rebuilt with numpy reshapes, numpy's float64 matmul, and the
Higham error bound.  See DESIGN.md "Oracle pins" (P1..P15).
"""
from __future__ import annotations

import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from tests.helpers import exact_product, gamma, stored_shape, unpack, unpack_op

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TRANS = ["NN", "NT", "TN", "TT"]


def run(tA, tB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, batch=1, sA=None, sB=None, sC=None):
    ra, ca = stored_shape(tA, M, K)
    rb, cb = stored_shape(tB, K, N)
    sA = lda * ca if sA is None else sA
    sB = ldb * cb if sB is None else sB
    sC = ldc * N if sC is None else sC
    return oracle.ref_gemm(tA, tB, M, N, K, alpha, A, lda, sA, B, ldb, sB, beta, C, ldc, sC, batch)


def col(*vals, dtype=np.float64):
    return np.array(vals, dtype=dtype)


# ---------------------------------------------------------------- P1..P3 hand cases
def test_p1_scalar_case():
    # SPEC.md:280 (simulator example): a=[2], b=[3], c=[5] -> 11
    ref, den, _ = run("N", "N", 1, 1, 1, 1.0, col(2.0), 1, col(3.0), 1, 1.0, col(5.0), 1)
    assert ref[0, 0, 0] == 11.0
    assert den[0, 0, 0] == 11.0


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_p2_identity(dtype):
    # alpha=1, beta=0, A=I3, B arbitrary -> C=B
    B = np.arange(1, 10, dtype=dtype)
    I3 = np.eye(3, dtype=dtype).ravel(order="F")
    ref, _, _ = run("N", "N", 3, 3, 3, 1.0, I3, 3, B, 3, 0.0, None, 3)
    assert np.array_equal(ref[0].ravel(), B.astype(np.float64))
    # A=[1,2;3,4] (column-major [1,3,2,4]), B=I2 -> C=A
    A = col(1, 3, 2, 4, dtype=dtype)
    I2 = np.eye(2, dtype=dtype).ravel(order="F")
    ref, _, _ = run("N", "N", 2, 2, 2, 1.0, A, 2, I2, 2, 0.0, None, 2)
    assert list(ref[0].ravel()) == [1, 3, 2, 4]


def test_p3_alpha_zero_scales_c():
    # alpha=0, beta=2, C=[1,2;3,4] -> [2,4;6,8]
    C = col(1, 3, 2, 4)
    nan = np.full(4, np.nan)
    ref, den, _ = run("N", "N", 2, 2, 2, 0.0, nan, 2, nan, 2, 2.0, C, 2)
    assert list(ref[0].ravel()) == [2, 6, 4, 8]
    assert list(den[0].ravel()) == [2, 6, 4, 8]


# ---------------------------------------------------------------- golden fixtures
def test_golden_worked_examples():
    with open(os.path.join(GOLDEN, "oracle_cases.json")) as f:
        cases = json.load(f)["cases"]
    assert cases
    for c in cases:
        ref, _, _ = run(c["transA"], c["transB"], c["M"], c["N"], c["K"], c["alpha"],
                        np.array(c["A"], dtype=np.float64), c["lda"],
                        np.array(c["B"], dtype=np.float64), c["ldb"], c["beta"],
                        np.array(c["C"], dtype=np.float64), c["ldc"])
        assert ref[0].ravel().tolist() == c["expect"], c["cite"]


# ---------------------------------------------------------------- P4 exact integers
ALPHAS = [-1.0, 0.0, 0.25, 0.5, 1.0, 1.5]


@pytest.mark.parametrize("tr", TRANS)
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_p4_integer_exact(tr, dtype):
    rng = np.random.default_rng(4)
    for M, N, K in [(5, 7, 80), (16, 16, 16), (1, 33, 9), (13, 2, 40)]:
        tA, tB = tr
        ra, ca = stored_shape(tA, M, K)
        rb, cb = stored_shape(tB, K, N)
        A = rng.integers(-8, 9, size=ra * ca).astype(dtype)
        B = rng.integers(-8, 9, size=rb * cb).astype(dtype)
        C = rng.integers(-8, 9, size=M * N).astype(dtype)
        prod = exact_product(unpack_op(A, 0, tA, M, K, ra), unpack_op(B, 0, tB, K, N, rb))
        for alpha, beta in itertools.product(ALPHAS, ALPHAS):
            ref, _, _ = run(tA, tB, M, N, K, alpha, A, ra, B, rb, beta, C, M)
            Cm = unpack(C, 0, M, N, M)
            for i, j in itertools.product(range(M), range(N)):
                want = Fraction(alpha) * prod[i, j] + Fraction(beta) * Fraction(float(Cm[i, j]))
                assert Fraction(ref[0, j, i]) == want


# ---------------------------------------------------------------- P5 permutations
@pytest.mark.parametrize("tB", ["N", "T"])
def test_p5_permutation(tB):
    rng = np.random.default_rng(5)
    M = K = 11
    N = 6
    perm = rng.permutation(M)
    P = np.zeros((M, K))
    P[np.arange(M), perm] = 1.0
    rb, cb = stored_shape(tB, K, N)
    B = rng.uniform(-1, 1, size=rb * cb)
    ref, _, _ = run("N", tB, M, N, K, 1.0, P.ravel(order="F"), M, B, rb, 0.0, None, M)
    opB = unpack_op(B, 0, tB, K, N, rb)
    # (P opB)(i, :) = opB(perm[i], :) exactly
    assert np.array_equal(ref[0].T, opB[perm, :])
    # columns: op(A) arbitrary, op(B) = permutation -> permuted columns of op(A)
    Q = np.zeros((K, N := K))
    permc = rng.permutation(K)
    Q[permc, np.arange(N)] = 1.0
    A = rng.uniform(-1, 1, size=M * K)
    ref, _, _ = run("N", "N", M, N, K, 1.0, A, M, Q.ravel(order="F"), K, 0.0, None, M)
    opA = unpack(A, 0, M, K, M)
    assert np.array_equal(ref[0].T, opA[:, permc])


# ---------------------------------------------------------------- P6 alpha/beta invariants
def test_p6_alpha_beta_invariants():
    rng = np.random.default_rng(6)
    M, N, K = 7, 5, 9
    A = rng.uniform(-1, 1, M * K)
    B = rng.uniform(-1, 1, K * N)
    C = rng.uniform(-1, 1, M * N)
    nanA = np.full(M * K, np.nan)
    nanB = np.full(K * N, np.nan)
    nanC = np.full(M * N, np.nan)
    # alpha=0, beta=1 -> C unchanged, A/B never read
    ref, _, _ = run("N", "N", M, N, K, 0.0, nanA, M, nanB, K, 1.0, C, M)
    assert np.array_equal(ref[0].ravel(), C)
    # alpha=0, beta=0 -> 0
    ref, _, _ = run("N", "N", M, N, K, 0.0, nanA, M, nanB, K, 0.0, nanC, M)
    assert np.all(ref == 0)
    # beta=0 with NaN C -> finite
    ref, den, _ = run("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, nanC, M)
    assert np.all(np.isfinite(ref)) and np.all(np.isfinite(den))
    # K = 0 -> C = beta*C
    ref, _, _ = run("N", "N", M, N, 0, 1.0, nanA, M, nanB, 1, 0.5, C, M)
    assert np.array_equal(ref[0].ravel(), 0.5 * C)


# ---------------------------------------------------------------- P7 transpose identity
@pytest.mark.parametrize("tr", TRANS)
def test_p7_transpose_identity(tr):
    # op(A)op(B) = (op(B)^T op(A)^T)^T : call (flip tB, flip tA, N, M, K, B, A)
    rng = np.random.default_rng(7)
    tA, tB = tr
    flip = {"N": "T", "T": "N"}
    M, N, K = 9, 13, 17
    ra, ca = stored_shape(tA, M, K)
    rb, cb = stored_shape(tB, K, N)
    A = rng.integers(-8, 9, ra * ca).astype(np.float64)
    B = rng.integers(-8, 9, rb * cb).astype(np.float64)
    ref1, _, _ = run(tA, tB, M, N, K, 1.0, A, ra, B, rb, 0.0, None, M)
    ref2, _, _ = run(flip[tB], flip[tA], N, M, K, 1.0, B, rb, A, ra, 0.0, None, N)
    assert np.array_equal(ref1[0], ref2[0].T)


# ---------------------------------------------------------------- P8 brute force 1..4^3
def dyadic(rng, n, dtype):
    # multiples of 2^-6 in [-1, 1]: every product/sum below is exact
    return (rng.integers(-64, 65, size=n) / 64.0).astype(dtype)


def test_p8_brute_force_small():
    rng = np.random.default_rng(8)
    ab = [0.0, 1.0, -1.0, 0.5]
    for M, N, K in itertools.product(range(1, 5), repeat=3):
        for tA, tB in TRANS:
            for pad in (0, 3):
                ra, ca = stored_shape(tA, M, K)
                rb, cb = stored_shape(tB, K, N)
                lda, ldb, ldc = ra + pad, rb + pad, M + pad
                batch = 2
                sA, sB, sC = lda * ca + pad, ldb * cb, ldc * N + 1
                A = np.full(batch * sA, np.nan)
                B = np.full(batch * sB, np.nan)
                C = np.full(batch * sC, np.nan)
                for b in range(batch):
                    for c in range(ca):
                        A[b * sA + c * lda:b * sA + c * lda + ra] = dyadic(rng, ra, np.float64)
                    for c in range(cb):
                        B[b * sB + c * ldb:b * sB + c * ldb + rb] = dyadic(rng, rb, np.float64)
                    for c in range(N):
                        C[b * sC + c * ldc:b * sC + c * ldc + M] = dyadic(rng, M, np.float64)
                prods = [exact_product(unpack_op(A, b * sA, tA, M, K, lda),
                                       unpack_op(B, b * sB, tB, K, N, ldb)) for b in range(batch)]
                for alpha, beta in itertools.product(ab, ab):
                    ref, _, _ = run(tA, tB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
                                    batch=batch, sA=sA, sB=sB, sC=sC)
                    assert np.all(np.isfinite(ref)), (M, N, K, tA, tB, pad)
                    for b in range(batch):
                        Cm = unpack(C, b * sC, M, N, ldc)
                        want = np.array([[float(Fraction(alpha) * prods[b][i, j] +
                                                Fraction(beta) * Fraction(float(Cm[i, j])))
                                          for j in range(N)] for i in range(M)])
                        assert np.array_equal(ref[b].T, want), (M, N, K, tA, tB, alpha, beta)


# ---------------------------------------------------------------- P9 numpy cross-check
@pytest.mark.parametrize("tr", TRANS)
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_p9_numpy_matmul(tr, dtype):
    rng = np.random.default_rng(9)
    tA, tB = tr
    M, N, K, batch = 19, 23, 31, 5
    ra, ca = stored_shape(tA, M, K)
    rb, cb = stored_shape(tB, K, N)
    A = rng.uniform(-1, 1, batch * ra * ca).astype(dtype)
    B = rng.uniform(-1, 1, batch * rb * cb).astype(dtype)
    C = rng.uniform(-1, 1, batch * M * N).astype(dtype)
    ref, _, _ = run(tA, tB, M, N, K, 1.5, A, ra, B, rb, 0.5, C, M, batch=batch)
    for b in range(batch):
        opA = unpack_op(A.astype(np.float64), b * ra * ca, tA, M, K, ra)
        opB = unpack_op(B.astype(np.float64), b * rb * cb, tB, K, N, rb)
        want = 1.5 * (opA @ opB) + 0.5 * unpack(C.astype(np.float64), b * M * N, M, N, M)
        np.testing.assert_allclose(ref[b].T, want, rtol=0, atol=1e-13)


# ---------------------------------------------------------------- P10 error bound
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_p10_error_bound_vs_exact(dtype):
    """|oracle - exact| <= gamma_K(2^-53) * den: the oracle's own error is far
    below the 1e-5 / 1e-13 parity tolerances, so a parity failure is a bug."""
    rng = np.random.default_rng(10)
    u = 2.0 ** -53
    for M, N, K in [(3, 4, 80), (2, 2, 64), (5, 1, 33)]:
        A = rng.uniform(-1, 1, M * K).astype(dtype)
        B = rng.uniform(-1, 1, K * N).astype(dtype)
        ref, den, _ = run("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, None, M)
        prod = exact_product(unpack(A, 0, M, K, M), unpack(B, 0, K, N, K))
        for i, j in itertools.product(range(M), range(N)):
            err = abs(Fraction(ref[0, j, i]) - prod[i, j])
            assert err <= Fraction(gamma(K, u) * 1.0001) * Fraction(den[0, j, i])
    # the tolerance arithmetic of DESIGN.md: fp32 FMA chain bound < 1e-5
    assert gamma(80, 2.0 ** -24) + 3 * 2.0 ** -24 < 1e-5
    assert gamma(80, 2.0 ** -53) * 2 + 6 * 2.0 ** -53 < 1e-13


# ---------------------------------------------------------------- P14 predicate
def test_p14_small_predicate():
    with open(os.path.join(GOLDEN, "predicate.json")) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        assert oracle.is_small(c["transA"], c["transB"], c["M"], c["N"], c["K"]) == c["small"], c


def test_max_rel_err_semantics():
    ref = np.array([1.0, 0.0, 2.0])
    den = np.array([1.0, 0.0, 1.0])
    assert oracle.max_rel_err(np.array([1.0, 0.0, 2.0]), ref, den) == 0.0
    assert oracle.max_rel_err(np.array([1.0, 1e-30, 2.0]), ref, den) == np.inf
    assert oracle.max_rel_err(np.array([1.0, 0.0, np.nan]), ref, den) == np.inf
    assert abs(oracle.max_rel_err(np.array([1.5, 0.0, 2.0]), ref, den) - 0.5) < 1e-15
