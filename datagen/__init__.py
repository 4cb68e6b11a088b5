"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it only turns
(seed, matrix id, global problem index, logical element index) into a value
uniform on [-1, 1), so that the CPU oracle and the GPU can each build the
same inputs independently.  It is imported by
tests/ and bench.py; neither oracle/ nor paper_2208_09822_b200/ imports it.

Counter-based generator (reading A15):
    ctr = ((seed*3 + mat) << 48) ^ (b*elems_per_problem + e)
    h   = splitmix64(ctr)       (Steele, Lea & Flood's 64-bit finaliser:
                                 z += 0x9E3779B97F4A7C15;
                                 z = (z ^ z>>30) * 0xBF58476D1CE4E5B9;
                                 z = (z ^ z>>27) * 0x94D049BB133111EB;
                                 z ^= z>>31)
    fp32: x = (h >> 40) * 2^-23 - 1       fp64: x = (h >> 11) * 2^-52 - 1
Both are exact, hence bit-identical on CPU (numpy, here) and GPU
(datagen/fill.cu, the CUDA twin).  mat: A=0, B=1, C=2.  b is the GLOBAL
problem index and e = r + c*rows the logical (ld-independent) element index.
Padding (ld > rows, stride > ld*cols) is filled with NaN sentinels so that any
read of it by the GEMM shows up in the result.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_CU = os.path.join(_HERE, "fill.cu")
_SO = os.path.join(_HERE, "libiaat_datagen.so")
MAT_A, MAT_B, MAT_C = 0, 1, 2

_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def values(seed: int, mat: int, dtype, ids, rows: int, cols: int) -> np.ndarray:
    """Logical values of matrices `ids` (global problem indices), shape
    (len(ids), cols, rows) -- column-major per problem, no padding."""
    ids = np.asarray(ids, dtype=np.uint64).reshape(-1, 1)
    epp = np.uint64(rows * cols)
    e = np.arange(rows * cols, dtype=np.uint64).reshape(1, -1)
    hi = np.uint64((seed * 3 + mat) & 0xFFFF) << np.uint64(48)
    with np.errstate(over="ignore"):
        ctr = hi ^ (ids * epp + e)
    h = splitmix64(ctr)
    if np.dtype(dtype) == np.float32:
        x = (h >> np.uint64(40)).astype(np.float64) * 2.0 ** -23 - 1.0
        x = x.astype(np.float32)
    else:
        x = (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -52 - 1.0
    return x.reshape(len(ids), cols, rows)


def fill_host(seed, mat, dtype, rows, cols, ld, stride, ids) -> np.ndarray:
    """Strided batch buffer for problems `ids` placed at local slots
    0..len(ids)-1: element (r, c) of slot s lives at s*stride + r + c*ld.
    Size = len(ids)*stride (at least ld*cols).  Padding = NaN."""
    n = len(ids)
    stride = max(stride, 0)
    size = max(n * stride, (n - 1) * stride + ld * cols if n else 0)
    buf = np.full(size, np.nan, dtype=dtype)
    v = values(seed, mat, dtype, ids, rows, cols)
    if rows == 0 or cols == 0 or n == 0:
        return buf
    slot = np.arange(n, dtype=np.int64).reshape(-1, 1, 1) * stride
    cc = np.arange(cols, dtype=np.int64).reshape(1, -1, 1) * ld
    rr = np.arange(rows, dtype=np.int64).reshape(1, 1, -1)
    buf[(slot + cc + rr).ravel()] = v.ravel()
    return buf


# ---------------------------------------------------------------- GPU twin
_lib = None


def build(force: bool = False, nvcc: str = "nvcc") -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_CU):
        tmp = _SO + ".tmp%d" % os.getpid()
        subprocess.check_call([nvcc, "-O3", "-gencode", "arch=compute_100a,code=sm_100a",
                               "-shared", "-Xcompiler", "-fPIC", "-o", tmp, _CU])
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        lib = ctypes.CDLL(_SO)
        i64 = ctypes.c_int64
        lib.iaat_datagen_fill.argtypes = [ctypes.c_int, i64, ctypes.c_int, i64, i64, i64,
                                          i64, i64, i64, ctypes.c_void_p, ctypes.c_void_p]
        lib.iaat_datagen_fill.restype = ctypes.c_int
        _lib = lib
    return _lib


def fill_device(t, seed, mat, rows, cols, ld, stride, batch, first_id=0, stream=None):
    """Fill torch CUDA tensor `t` (flat, float32/float64) with problems
    first_id .. first_id+batch-1 at local slots 0..batch-1 (NaN padding)."""
    import torch
    dt = {torch.float32: 0, torch.float64: 1}[t.dtype]
    need = (batch - 1) * stride + ld * cols if batch else 0
    assert t.numel() >= need, (t.numel(), need)
    if stream is None:
        stream = torch.cuda.current_stream().cuda_stream
    rc = _load().iaat_datagen_fill(dt, seed, mat, rows, cols, ld, stride, batch,
                                   first_id, ctypes.c_void_p(t.data_ptr()),
                                   ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError("iaat_datagen_fill failed: cuda error %d" % rc)
