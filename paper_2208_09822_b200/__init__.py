"""B200-native batched small GEMM (IAAT, arXiv 2208.09822, re-designed for sm_100a).

The product is libiaat.so (C ABI: include/iaat.h); `iaat` is its ctypes
binding.  Build with `python -m paper_2208_09822_b200.build`.  The binding is
loaded on first use of any of its names (so that the build module can run
before the library exists); without libiaat.so that first use fails loudly --
there is no CPU fallback.
"""
_NAMES = (
    "IAAT_R32F", "IAAT_R64F", "IAAT_C32F", "IAAT_C64F", "IaatError", "gemm_batched", "gemm_strided_batched",
    "iaat_catalog_describe", "iaat_gemm_batched", "iaat_gemm_grouped_strided", "iaat_gemm_strided_batched", "iaat_is_small_gemm",
    "iaat_last_cuda_error", "iaat_launch_count", "iaat_paper_tile", "iaat_plan_describe", "iaat_status_string",
    "iaat_set_tn_limit", "iaat_get_tn_limit",
    "iaat_version",
)


def __getattr__(name):
    if name in _NAMES:
        from . import iaat
        return getattr(iaat, name)
    raise AttributeError(name)
