"""Test helpers that are independent of both the oracle and the CUDA path.

`unpack_op` rebuilds op(X) as a dense matrix with numpy reshapes/transposes
(library routines), NOT with the oracle's index formulas, so that comparing
the oracle with `exact_product` really pins the oracle's indexing.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np


def stored_shape(trans, rows_op, cols_op):
    """Stored (rows, cols) of X when op(X) is rows_op x cols_op."""
    return (rows_op, cols_op) if trans in "Nn" else (cols_op, rows_op)


def unpack(buf, off, rows, cols, ld):
    """Dense rows x cols column-major matrix stored at buf[off] with ld."""
    if rows == 0 or cols == 0:
        return np.zeros((rows, cols), dtype=buf.dtype)
    # pad the flat slice so that reshape(cols, ld) is always possible
    need = ld * cols
    sl = buf[off:off + need]
    if sl.size < need:
        sl = np.concatenate([sl, np.full(need - sl.size, np.nan, dtype=buf.dtype)])
    return sl.reshape(cols, ld).T[:rows, :]


def unpack_op(buf, off, trans, rows_op, cols_op, ld):
    r, c = stored_shape(trans, rows_op, cols_op)
    X = unpack(buf, off, r, c, ld)
    return X if trans in "Nn" else X.T


def to_frac(X):
    out = np.empty(X.shape, dtype=object)
    for idx, v in np.ndenumerate(X):
        out[idx] = Fraction(float(v))
    return out


def exact_product(opA, opB):
    """Exact rational op(A) @ op(B) (object-dtype matmul of Fractions)."""
    M, K = opA.shape
    K2, N = opB.shape
    assert K == K2
    if K == 0:
        out = np.empty((M, N), dtype=object)
        out.fill(Fraction(0))
        return out
    return to_frac(opA).dot(to_frac(opB))


def gamma(n, u):
    return n * u / (1 - n * u)
