"""B200-native batched small GEMM (IAAT, arXiv 2208.09822, re-designed for sm_100a).

The product is libiaat.so (C ABI: include/iaat.h); `iaat` is its ctypes
binding.  Build with `python -m paper_2208_09822_b200.build`.
"""
from .iaat import (  # noqa: F401
    IAAT_R32F, IAAT_R64F, IaatError, gemm_batched, gemm_strided_batched, iaat_catalog_describe,
    iaat_gemm_batched, iaat_gemm_strided_batched, iaat_is_small_gemm, iaat_last_cuda_error,
    iaat_launch_count, iaat_plan_describe, iaat_status_string, iaat_version,
)
