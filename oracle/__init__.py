"""CPU oracle for batched small GEMM -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2208_09822_b200``) never imports it, and this package
imports nothing from the product path.

The arithmetic lives in ``oracle/ref_gemm.c`` (plain C triple loop, fp64
accumulation, k ascending; Sec. I "C = alpha A x B + beta C",
PAPER.md:101 Table I note "NT means A is not transposed and B transposed ...
column-major").  This module only loads it with ctypes and marshals numpy
arrays.

Parity status: pinned (tests/test_oracle_pins.py: hand cases, exact integer
results vs Python Fractions, identity/permutation, alpha/beta invariants,
transpose identity, brute force 1..4^3, numpy float64 cross-check, ld padding
with NaN sentinels, the Higham error bound).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ref_gemm.c")
_LIB = os.path.join(_HERE, "libiaat_oracle.so")
_lib = None

GCC_FLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-shared", "-fPIC", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile ref_gemm.c with gcc (no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", *GCC_FLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i64, dbl, vp = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
        lib.iaat_ref_gemm.argtypes = [
            ctypes.c_int, ctypes.c_char, ctypes.c_char, i64, i64, i64, dbl,
            vp, i64, i64, vp, i64, i64, dbl, vp, i64, i64, i64, vp, vp,
            ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        lib.iaat_ref_gemm.restype = ctypes.c_int
        dp = ctypes.POINTER(ctypes.c_double)
        lib.iaat_ref_cgemm.argtypes = [
            ctypes.c_int, ctypes.c_char, ctypes.c_char, i64, i64, i64, dp,
            vp, i64, i64, vp, i64, i64, dp, vp, i64, i64, i64, vp, vp,
            ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        lib.iaat_ref_cgemm.restype = ctypes.c_int
        lib.iaat_ref_is_small.argtypes = [ctypes.c_char, ctypes.c_char, i64, i64, i64]
        lib.iaat_ref_is_small.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def ref_gemm(transA, transB, M, N, K, alpha, A, lda, strideA, B, ldb, strideB,
             beta, C, ldc, strideC, batch, nthreads: int = 0, want_den=True):
    """Reference C = alpha*op(A)op(B) + beta*C for `batch` problems.

    A, B, C are flat numpy arrays (float32 or float64, same dtype) holding the
    whole batch at the given element strides.  Returns (ref, den, threads)
    where ref/den are float64 arrays of shape (batch, N, M) -- i.e. each
    problem packed column-major (ref[b, j, i] = C_b(i, j)).
    """
    A = np.ascontiguousarray(A)
    B = np.ascontiguousarray(B)
    dtype = {np.dtype(np.float32): 0, np.dtype(np.float64): 1}[A.dtype]
    assert B.dtype == A.dtype
    if C is not None:
        C = np.ascontiguousarray(C)
        assert C.dtype == A.dtype
    ref = np.empty((batch, N, M), dtype=np.float64)
    den = np.empty((batch, N, M), dtype=np.float64) if want_den else None
    used = ctypes.c_int(0)
    rc = _load().iaat_ref_gemm(
        dtype, transA.encode(), transB.encode(), M, N, K, float(alpha),
        _ptr(A), lda, strideA, _ptr(B), ldb, strideB, float(beta),
        _ptr(C) if (C is not None and beta != 0) else None, ldc, strideC, batch,
        _ptr(ref), _ptr(den), int(nthreads), ctypes.byref(used))
    if rc != 0:
        raise ValueError("iaat_ref_gemm rejected its arguments")
    return ref, den, used.value


def ref_cgemm(transA, transB, M, N, K, alpha, A, lda, strideA, B, ldb, strideB,
              beta, C, ldc, strideC, batch, nthreads: int = 0, want_den=True):
    """Complex reference (CGEMM / ZGEMM): A, B, C flat complex64 / complex128
    numpy arrays (interleaved re, im), ld's and strides in complex elements,
    alpha / beta Python complex.  Returns (ref, den, threads): ref complex128
    of shape (batch, N, M), den float64 (batch, N, M) with the 1-norm bound
    of oracle/ref_gemm.c."""
    A = np.ascontiguousarray(A)
    B = np.ascontiguousarray(B)
    dtype = {np.dtype(np.complex64): 2, np.dtype(np.complex128): 3}[A.dtype]
    assert B.dtype == A.dtype
    alpha, beta = complex(alpha), complex(beta)
    if C is not None:
        C = np.ascontiguousarray(C)
        assert C.dtype == A.dtype
    ref = np.empty((batch, N, M), dtype=np.complex128)
    den = np.empty((batch, N, M), dtype=np.float64) if want_den else None
    al = (ctypes.c_double * 2)(alpha.real, alpha.imag)
    be = (ctypes.c_double * 2)(beta.real, beta.imag)
    used = ctypes.c_int(0)
    rc = _load().iaat_ref_cgemm(
        dtype, transA.encode(), transB.encode(), M, N, K, al,
        _ptr(A), lda, strideA, _ptr(B), ldb, strideB, be,
        _ptr(C) if (C is not None and beta != 0) else None, ldc, strideC, batch,
        _ptr(ref), _ptr(den), int(nthreads), ctypes.byref(used))
    if rc != 0:
        raise ValueError("iaat_ref_cgemm rejected its arguments")
    return ref, den, used.value


def max_rel_err_complex(got, ref, den):
    """Complex normalised error: max over elements of
    max(|re(got - ref)|, |im(got - ref)|) / den (den: the 1-norm bound)."""
    got = np.asarray(got, dtype=np.complex128)
    d = np.maximum(np.abs(got.real - ref.real), np.abs(got.imag - ref.imag))
    bad = (np.isnan(got.real) | np.isnan(got.imag)) & ~(np.isnan(ref.real) | np.isnan(ref.imag))
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(den > 0, d / np.where(den > 0, den, 1.0), np.where(d == 0, 0.0, np.inf))
    rel = np.where(bad, np.inf, rel)
    return float(rel.max()) if rel.size else 0.0


def is_small(transA, transB, M, N, K) -> bool:
    """PAPER.md:36 small-GEMM predicate (integer form, reading A10)."""
    return bool(_load().iaat_ref_is_small(transA.encode(), transB.encode(), M, N, K))


def max_rel_err(got_packed, ref, den):
    """Normalised error of north_star: |got - ref| / den elementwise, max.

    Where den == 0 the result must equal ref exactly (returns inf otherwise).
    NaN anywhere in `got` where ref is finite is an infinite error.
    """
    got = np.asarray(got_packed, dtype=np.float64)
    diff = np.abs(got - ref)
    bad_nan = np.isnan(got) & ~np.isnan(ref)
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(den > 0, diff / np.where(den > 0, den, 1.0),
                       np.where(diff == 0, 0.0, np.inf))
    rel = np.where(bad_nan, np.inf, rel)
    return float(rel.max()) if rel.size else 0.0
