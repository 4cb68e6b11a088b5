"""Thin ctypes binding of include/iaat.h (argument marshalling only).

Every name mirrors the C ABI.  No arithmetic happens here: each call goes
straight into libiaat.so, which enqueues sm_100a kernels or returns an error
status.  If the library is missing the import fails loudly -- there is no
CPU fallback.  Torch is used only to obtain device pointers and the current
stream in the convenience wrappers at the bottom.
"""
from __future__ import annotations

import ctypes
import json
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libiaat.so")

IAAT_R32F, IAAT_R64F, IAAT_C32F, IAAT_C64F = 0, 1, 2, 3
STATUS = {
    0: "IAAT_SUCCESS",
    1: "IAAT_ERROR_INVALID_VALUE",
    2: "IAAT_ERROR_NOT_SMALL",
    3: "IAAT_ERROR_ARCH",
    4: "IAAT_ERROR_CUDA",
    5: "IAAT_ERROR_NOT_SUPPORTED",
}

# exported symbols of include/iaat.h (tests check the .so exports exactly these)
EXPORTS = [
    "iaat_gemm_strided_batched", "iaat_gemm_batched",
    "iaat_sgemm_strided_batched", "iaat_dgemm_strided_batched",
    "iaat_sgemm_batched", "iaat_dgemm_batched",
    "iaat_cgemm_strided_batched", "iaat_zgemm_strided_batched", "iaat_gemm_grouped_strided",
    "iaat_is_small_gemm", "iaat_set_tn_limit", "iaat_get_tn_limit", "iaat_plan_describe", "iaat_catalog_describe", "iaat_paper_tile",
    "iaat_status_string", "iaat_last_cuda_error", "iaat_launch_count", "iaat_version",
]


class IaatError(RuntimeError):
    def __init__(self, status, what=""):
        self.status = status
        super().__init__("%s%s" % (STATUS.get(status, status), (": " + what) if what else ""))


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError("libiaat.so not built (%s): run `python -m paper_2208_09822_b200.build` "
                          "-- there is no CPU fallback" % LIB_PATH)
    lib = ctypes.CDLL(LIB_PATH)
    i64, vp, c, i = ctypes.c_int64, ctypes.c_void_p, ctypes.c_char, ctypes.c_int
    lib.iaat_gemm_strided_batched.argtypes = [i, c, c, i64, i64, i64, vp, vp, i64, i64, vp, i64, i64,
                                              vp, vp, i64, i64, i64, vp]
    lib.iaat_gemm_strided_batched.restype = i
    lib.iaat_gemm_batched.argtypes = [i, c, c, i64, i64, i64, vp, vp, i64, vp, i64, vp, vp, i64, i64, vp]
    lib.iaat_gemm_batched.restype = i
    lib.iaat_is_small_gemm.argtypes = [c, c, i64, i64, i64]
    lib.iaat_is_small_gemm.restype = i
    lib.iaat_set_tn_limit.argtypes = [i64]
    lib.iaat_set_tn_limit.restype = i
    lib.iaat_get_tn_limit.restype = i64
    lib.iaat_plan_describe.argtypes = [i, c, c, i64, i64, i64, i64, i64, i64, i64, i64, i64, i64, i, i,
                                       i64, i, ctypes.c_char_p, ctypes.c_size_t]
    lib.iaat_plan_describe.restype = i
    P = ctypes.POINTER
    lib.iaat_gemm_grouped_strided.argtypes = [i, i64, ctypes.c_char_p, ctypes.c_char_p, P(i64), P(i64), P(i64),
                                              vp, P(vp), P(i64), P(i64), P(vp), P(i64), P(i64), vp, P(vp),
                                              P(i64), P(i64), P(i64), vp]
    lib.iaat_gemm_grouped_strided.restype = i
    lib.iaat_paper_tile.argtypes = [i, i64, i64, ctypes.c_char_p, ctypes.c_size_t]
    lib.iaat_paper_tile.restype = i
    lib.iaat_catalog_describe.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
    lib.iaat_catalog_describe.restype = i
    lib.iaat_status_string.argtypes = [i]
    lib.iaat_status_string.restype = ctypes.c_char_p
    lib.iaat_last_cuda_error.restype = i
    lib.iaat_launch_count.restype = i64
    lib.iaat_version.restype = i
    return lib


_lib = _load()


def _ch(x):
    return x.encode() if isinstance(x, str) else bytes([x]) if isinstance(x, int) else x


def _scalar(dtype, v):
    """Host scalar of the call's dtype; complex dtypes take (re, im) pairs."""
    if dtype == IAAT_C32F:
        v = complex(v)
        return (ctypes.c_float * 2)(v.real, v.imag)
    if dtype == IAAT_C64F:
        v = complex(v)
        return (ctypes.c_double * 2)(v.real, v.imag)
    return ctypes.byref(ctypes.c_float(v) if dtype == IAAT_R32F else ctypes.c_double(v))


# ---------------------------------------------------------------- C-ABI mirrors
def iaat_gemm_strided_batched(dtype, transA, transB, M, N, K, alpha, A, lda, strideA, B, ldb, strideB,
                              beta, C, ldc, strideC, batch, stream=0):
    """A, B, C, stream: integer device addresses / cudaStream_t.  alpha,
    beta: Python floats (passed as host scalars of `dtype`).  Returns status."""
    return _lib.iaat_gemm_strided_batched(dtype, _ch(transA), _ch(transB), M, N, K, _scalar(dtype, alpha),
                                          A, lda, strideA, B, ldb, strideB, _scalar(dtype, beta), C, ldc,
                                          strideC, batch, stream)


def iaat_gemm_batched(dtype, transA, transB, M, N, K, alpha, Aarray, lda, Barray, ldb, beta, Carray, ldc,
                      batch, stream=0):
    """Aarray/Barray/Carray: integer DEVICE addresses of device pointer arrays."""
    return _lib.iaat_gemm_batched(dtype, _ch(transA), _ch(transB), M, N, K, _scalar(dtype, alpha), Aarray,
                                  lda, Barray, ldb, _scalar(dtype, beta), Carray, ldc, batch, stream)


def iaat_is_small_gemm(transA, transB, M, N, K) -> bool:
    return bool(_lib.iaat_is_small_gemm(_ch(transA), _ch(transB), M, N, K))


def iaat_set_tn_limit(max_mnk) -> int:
    """Raise (or restore) the TN domain bound M*N*K <= max_mnk, 32768..512000."""
    return _lib.iaat_set_tn_limit(max_mnk)


def iaat_get_tn_limit() -> int:
    return _lib.iaat_get_tn_limit()


def iaat_plan_describe(dtype, transA, transB, M, N, K, lda, strideA, ldb, strideB, ldc, strideC, batch,
                       beta_is_zero=False, alpha_is_zero=False, base_align_bytes=256, sm_count=148):
    buf = ctypes.create_string_buffer(16384)
    st = _lib.iaat_plan_describe(dtype, _ch(transA), _ch(transB), M, N, K, lda, strideA, ldb, strideB, ldc,
                                 strideC, batch, int(beta_is_zero), int(alpha_is_zero), base_align_bytes,
                                 sm_count, buf, len(buf))
    if st != 0:
        raise IaatError(st, "iaat_plan_describe")
    return json.loads(buf.value.decode())


def iaat_gemm_grouped_strided(dtype, groups, stream=0):
    """groups: list of dicts with keys transA, transB, M, N, K, alpha, A, lda,
    strideA, B, ldb, strideB, beta, C, ldc, strideC, batch (A/B/C integer
    device addresses).  Marshals the host arrays of the C ABI; returns status."""
    n = len(groups)
    i64a = lambda key: (ctypes.c_int64 * max(n, 1))(*[int(g[key]) for g in groups])  # noqa: E731
    ptra = lambda key: (ctypes.c_void_p * max(n, 1))(*[g[key] for g in groups])  # noqa: E731
    if dtype in (IAAT_C32F, IAAT_C64F):
        ct = ctypes.c_float if dtype == IAAT_C32F else ctypes.c_double
        flat = lambda key: (ct * max(2 * n, 1))(*[x for g in groups for x in (complex(g[key]).real,  # noqa: E731
                                                                                 complex(g[key]).imag)])
    else:
        ct = ctypes.c_float if dtype == IAAT_R32F else ctypes.c_double
        flat = lambda key: (ct * max(n, 1))(*[float(g[key]) for g in groups])  # noqa: E731
    ta = "".join(g["transA"] for g in groups).encode()
    tb = "".join(g["transB"] for g in groups).encode()
    return _lib.iaat_gemm_grouped_strided(dtype, n, ta, tb, i64a("M"), i64a("N"), i64a("K"), flat("alpha"),
                                          ptra("A"), i64a("lda"), i64a("strideA"), ptra("B"), i64a("ldb"),
                                          i64a("strideB"), flat("beta"), ptra("C"), i64a("ldc"), i64a("strideC"),
                                          i64a("batch"), stream)


def iaat_paper_tile(mode, M, N):
    """Paper-faithful SGEMM_NN tiling (mode 0 Alg. 2 literal, 1 optimum over Table I)."""
    buf = ctypes.create_string_buffer(1 << 16)
    st = _lib.iaat_paper_tile(mode, M, N, buf, len(buf))
    if st != 0:
        raise IaatError(st, "iaat_paper_tile")
    return json.loads(buf.value.decode())


def iaat_catalog_describe():
    buf = ctypes.create_string_buffer(1 << 20)
    st = _lib.iaat_catalog_describe(buf, len(buf))
    if st != 0:
        raise IaatError(st, "iaat_catalog_describe")
    return json.loads(buf.value.decode())


def iaat_status_string(status) -> str:
    return _lib.iaat_status_string(status).decode()


def iaat_last_cuda_error() -> int:
    return _lib.iaat_last_cuda_error()


def iaat_launch_count() -> int:
    return _lib.iaat_launch_count()


def iaat_version() -> int:
    return _lib.iaat_version()


# ---------------------------------------------------------------- torch convenience
def _stream_handle(stream):
    import torch
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def gemm_strided_batched(transA, transB, M, N, K, alpha, A, lda, strideA, B, ldb, strideB, beta, C, ldc,
                         strideC, batch, stream=None, check=True):
    """Same call with torch CUDA tensors (float32 or float64, flat or any
    shape; only data_ptr() is used).  Raises IaatError on a non-success
    status when check=True."""
    import torch
    dtype = {torch.float32: IAAT_R32F, torch.float64: IAAT_R64F, torch.complex64: IAAT_C32F,
             torch.complex128: IAAT_C64F}[C.dtype]
    st = iaat_gemm_strided_batched(dtype, transA, transB, M, N, K, alpha, A.data_ptr(), lda, strideA,
                                   B.data_ptr(), ldb, strideB, beta, C.data_ptr(), ldc, strideC, batch,
                                   _stream_handle(stream))
    if check and st != 0:
        raise IaatError(st, "cuda error %d" % iaat_last_cuda_error() if st == 4 else "")
    return st


def gemm_batched(transA, transB, M, N, K, alpha, Aptrs, lda, Bptrs, ldb, beta, Cptrs, ldc, batch,
                 dtype, stream=None, check=True):
    """Aptrs/Bptrs/Cptrs: int64 CUDA tensors holding device addresses."""
    st = iaat_gemm_batched(dtype, transA, transB, M, N, K, alpha, Aptrs.data_ptr(), lda, Bptrs.data_ptr(),
                           ldb, beta, Cptrs.data_ptr(), ldc, batch, _stream_handle(stream))
    if check and st != 0:
        raise IaatError(st, "cuda error %d" % iaat_last_cuda_error() if st == 4 else "")
    return st
