"""Pins for the complex oracle (oracle/ref_gemm.c iaat_ref_cgemm; SURVEY f1:
CGEMM / ZGEMM, Table I, Eq. 2) -- CPU only.

Checked against things other than itself: the already-pinned real oracle
(complex inputs with zero imaginary parts, and purely imaginary A), exact
Gaussian-integer / dyadic arithmetic on dense matrices rebuilt with numpy
reshapes (Python Fractions, independent of the oracle's index formulas),
numpy complex128 matmul, algebraic identities (alpha = i rotates, transpose
identity) and the error bound.
"""
from __future__ import annotations

import itertools
from fractions import Fraction

import numpy as np
import pytest

import oracle
from tests.helpers import gamma, stored_shape, unpack, unpack_op

TRANS = ["NN", "NT", "TN", "TT"]
CDT = [np.complex64, np.complex128]


def crun(tA, tB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, batch=1, sA=None, sB=None, sC=None):
    ra, ca = stored_shape(tA, M, K)
    rb, cb = stored_shape(tB, K, N)
    sA = lda * ca if sA is None else sA
    sB = ldb * cb if sB is None else sB
    sC = ldc * N if sC is None else sC
    return oracle.ref_cgemm(tA, tB, M, N, K, alpha, A, lda, sA, B, ldb, sB, beta, C, ldc, sC, batch)


def gauss_dyadic(rng, n, dtype):
    """Complex entries with integer/4 parts in [-2, 2]: every product and
    sum below stays exactly representable (small dyadic rationals)."""
    re = rng.integers(-8, 9, size=n) / 4.0
    im = rng.integers(-8, 9, size=n) / 4.0
    return (re + 1j * im).astype(dtype)


def frac_c(z):
    return (Fraction(float(z.real)), Fraction(float(z.imag)))


def cmul(x, y):
    return (x[0] * y[0] - x[1] * y[1], x[0] * y[1] + x[1] * y[0])


def cadd(x, y):
    return (x[0] + y[0], x[1] + y[1])


def exact_cproduct(opA, opB):
    M, K = opA.shape
    N = opB.shape[1]
    out = np.empty((M, N), dtype=object)
    for i in range(M):
        for j in range(N):
            s = (Fraction(0), Fraction(0))
            for k in range(K):
                s = cadd(s, cmul(frac_c(opA[i, k]), frac_c(opB[k, j])))
            out[i, j] = s
    return out


@pytest.mark.parametrize("tr", TRANS)
@pytest.mark.parametrize("dt", [(np.complex64, np.float32), (np.complex128, np.float64)])
def test_zero_imaginary_reduces_to_real_oracle(tr, dt):
    """Real inputs embedded in C: the complex oracle equals the (pinned) real
    oracle bitwise, including the error denominator."""
    cdt, rdt = dt
    rng = np.random.default_rng(1)
    M, N, K, b = 5, 7, 9, 3
    ra, ca = stored_shape(tr[0], M, K)
    rb, cb = stored_shape(tr[1], K, N)
    Ar = rng.uniform(-1, 1, ra * ca * b).astype(rdt)
    Br = rng.uniform(-1, 1, rb * cb * b).astype(rdt)
    Cr = rng.uniform(-1, 1, M * N * b).astype(rdt)
    ref_r, den_r, _ = oracle.ref_gemm(tr[0], tr[1], M, N, K, 1.5, Ar, ra, ra * ca, Br, rb, rb * cb, -0.5, Cr, M,
                                      M * N, b)
    ref_c, den_c, _ = oracle.ref_cgemm(tr[0], tr[1], M, N, K, 1.5, Ar.astype(cdt), ra, ra * ca, Br.astype(cdt),
                                       rb, rb * cb, -0.5, Cr.astype(cdt), M, M * N, b)
    assert np.array_equal(ref_c.real, ref_r)
    assert np.all(ref_c.imag == 0)
    assert np.array_equal(den_c, den_r)


def test_imaginary_a_rotates_result():
    """A = i*X with X real, B real, alpha = 1, beta = 0: the result is i times
    the real product -- real part exactly 0, imaginary part bitwise the real
    oracle's."""
    rng = np.random.default_rng(2)
    M, N, K = 6, 4, 11
    X = rng.uniform(-1, 1, M * K)
    Y = rng.uniform(-1, 1, K * N)
    ref_r, _, _ = oracle.ref_gemm("N", "N", M, N, K, 1.0, X, M, M * K, Y, K, K * N, 0.0, None, M, M * N, 1)
    ref_c, _, _ = oracle.ref_cgemm("N", "N", M, N, K, 1.0, 1j * X, M, M * K, Y.astype(np.complex128), K, K * N,
                                   0.0, None, M, M * N, 1)
    assert np.all(ref_c.real == 0)
    assert np.array_equal(ref_c.imag, ref_r)


@pytest.mark.parametrize("tr", TRANS)
@pytest.mark.parametrize("cdt", CDT)
def test_gaussian_dyadic_exact(tr, cdt):
    """Dyadic complex entries (exact in fp32 and fp64), K up to 40, complex
    alpha/beta from a dyadic grid: the oracle equals exact rational complex
    arithmetic bitwise (all intermediates are exactly representable)."""
    rng = np.random.default_rng(3)
    for (M, N, K) in ((1, 1, 1), (3, 5, 7), (8, 4, 40), (13, 11, 2)):
        ra, ca = stored_shape(tr[0], M, K)
        rb, cb = stored_shape(tr[1], K, N)
        A = gauss_dyadic(rng, ra * ca, cdt)
        B = gauss_dyadic(rng, rb * cb, cdt)
        C = gauss_dyadic(rng, M * N, cdt)
        P = exact_cproduct(unpack_op(A, 0, tr[0], M, K, ra), unpack_op(B, 0, tr[1], K, N, rb))
        Cm = unpack(C, 0, M, N, M)
        for alpha, beta in ((1, 0), (0.5 - 1j, 0), (1j, 0.25 + 0.75j), (-1, 1), (0, 2j)):
            ref, _, _ = crun(tr[0], tr[1], M, N, K, alpha, A, ra, B, rb, beta, C, M)
            al = (Fraction(alpha.real if isinstance(alpha, complex) else alpha),
                  Fraction(alpha.imag if isinstance(alpha, complex) else 0))
            be = (Fraction(complex(beta).real), Fraction(complex(beta).imag))
            for i in range(M):
                for j in range(N):
                    want = cmul(al, P[i, j]) if (alpha != 0) else (Fraction(0), Fraction(0))
                    if beta != 0:
                        want = cadd(want, cmul(be, frac_c(Cm[i, j])))
                    got = ref[0, j, i]
                    assert got.real == float(want[0]) and got.imag == float(want[1]), (tr, M, N, K, alpha, beta)


def test_brute_force_small_with_padding():
    """All (M,N,K) in {1..3}^3 x 4 transpositions, ld = min + 2 with NaN
    padding and gaps between problems, alpha/beta in {0, 1, i, -0.5}: exact
    complex rationals built from numpy reshapes."""
    rng = np.random.default_rng(4)
    ab = [0, 1, 1j, -0.5]
    for M, N, K in itertools.product(range(1, 4), repeat=3):
        for tA, tB in TRANS:
            pad = 2
            ra, ca = stored_shape(tA, M, K)
            rb, cb = stored_shape(tB, K, N)
            lda, ldb, ldc = ra + pad, rb + pad, M + pad
            batch = 2
            sA, sB, sC = lda * ca + 1, ldb * cb + 1, ldc * N + 1
            nan = complex(np.nan, np.nan)
            A = np.full(batch * sA, nan, dtype=np.complex128)
            B = np.full(batch * sB, nan, dtype=np.complex128)
            C = np.full(batch * sC, nan, dtype=np.complex128)
            for b in range(batch):
                for c in range(ca):
                    A[b * sA + c * lda:b * sA + c * lda + ra] = gauss_dyadic(rng, ra, np.complex128)
                for c in range(cb):
                    B[b * sB + c * ldb:b * sB + c * ldb + rb] = gauss_dyadic(rng, rb, np.complex128)
                for c in range(N):
                    C[b * sC + c * ldc:b * sC + c * ldc + M] = gauss_dyadic(rng, M, np.complex128)
            prods = [exact_cproduct(unpack_op(A, b * sA, tA, M, K, lda), unpack_op(B, b * sB, tB, K, N, ldb))
                     for b in range(batch)]
            for alpha, beta in itertools.product(ab, ab):
                ref, _, _ = crun(tA, tB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, batch=batch, sA=sA,
                                 sB=sB, sC=sC)
                assert np.all(np.isfinite(ref)), (M, N, K, tA, tB)
                al = (Fraction(complex(alpha).real), Fraction(complex(alpha).imag))
                be = (Fraction(complex(beta).real), Fraction(complex(beta).imag))
                for b in range(batch):
                    Cm = unpack(C, b * sC, M, N, ldc)
                    for i in range(M):
                        for j in range(N):
                            want = cmul(al, prods[b][i, j]) if alpha != 0 else (Fraction(0), Fraction(0))
                            if beta != 0:
                                want = cadd(want, cmul(be, frac_c(Cm[i, j])))
                            z = ref[b, j, i]
                            assert (z.real, z.imag) == (float(want[0]), float(want[1])), (M, N, K, tA, tB)


@pytest.mark.parametrize("tr", TRANS)
@pytest.mark.parametrize("cdt", CDT)
def test_numpy_complex_matmul(tr, cdt):
    rng = np.random.default_rng(5)
    M, N, K, b = 9, 12, 17, 4
    ra, ca = stored_shape(tr[0], M, K)
    rb, cb = stored_shape(tr[1], K, N)
    A = (rng.uniform(-1, 1, ra * ca * b) + 1j * rng.uniform(-1, 1, ra * ca * b)).astype(cdt)
    B = (rng.uniform(-1, 1, rb * cb * b) + 1j * rng.uniform(-1, 1, rb * cb * b)).astype(cdt)
    C = (rng.uniform(-1, 1, M * N * b) + 1j * rng.uniform(-1, 1, M * N * b)).astype(cdt)
    alpha, beta = 0.75 - 0.5j, -1.25 + 2j
    ref, den, _ = crun(tr[0], tr[1], M, N, K, alpha, A, ra, B, rb, beta, C, M, batch=b)
    for q in range(b):
        oa = unpack_op(A, q * ra * ca, tr[0], M, K, ra).astype(np.complex128)
        ob = unpack_op(B, q * rb * cb, tr[1], K, N, rb).astype(np.complex128)
        cm = unpack(C, q * M * N, M, N, M).astype(np.complex128)
        want = alpha * (oa @ ob) + beta * cm
        assert np.max(np.abs(ref[q].T - want) / den[q].T) < 1e-14


def test_transpose_identity_and_error_bound():
    """op(A)op(B) = (op(B)^T op(A)^T)^T (exact for dyadic entries); and on
    random fp32 complex data |oracle - exact| <= gamma_2K(2^-53) * den."""
    rng = np.random.default_rng(6)
    M, N, K = 7, 5, 13
    A = gauss_dyadic(rng, M * K, np.complex128)
    B = gauss_dyadic(rng, K * N, np.complex128)
    r1, _, _ = crun("N", "N", M, N, K, 1 - 1j, A, M, B, K, 0, None, M)
    r2, _, _ = crun("T", "T", N, M, K, 1 - 1j, B, K, A, M, 0, None, N)
    assert np.array_equal(r1[0], r2[0].T)
    A = (rng.uniform(-1, 1, M * K) + 1j * rng.uniform(-1, 1, M * K)).astype(np.complex64)
    B = (rng.uniform(-1, 1, K * N) + 1j * rng.uniform(-1, 1, K * N)).astype(np.complex64)
    ref, den, _ = crun("N", "N", M, N, K, 1, A, M, B, K, 0, None, M)
    P = exact_cproduct(unpack_op(A, 0, "N", M, K, M), unpack_op(B, 0, "N", K, N, K))
    g = gamma(2 * K + 2, 2.0 ** -53)
    for i in range(M):
        for j in range(N):
            z = ref[0, j, i]
            assert abs(Fraction(float(z.real)) - P[i, j][0]) <= Fraction(g) * Fraction(float(den[0, j, i]))
            assert abs(Fraction(float(z.imag)) - P[i, j][1]) <= Fraction(g) * Fraction(float(den[0, j, i]))
