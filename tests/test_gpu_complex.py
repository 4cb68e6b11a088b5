"""GPU parity of the complex path (CGEMM / ZGEMM) against the
complex oracle, through the C ABI.  Tolerance: with the 1-norm
denominator every real component is one FMA chain of length 2K (plus the
alpha/beta epilogue), so |err| <= (gamma_2K + 4u) den: fp32 K <= 80 ->
9.8e-6 < 1e-5; fp64 < 1e-13."""
from __future__ import annotations

import itertools

import numpy as np
import pytest

from tests.gpu_utils import CCase, sample_ids

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TRANS = ["NN", "NT", "TN", "TT"]
CDT = [np.complex64, np.complex128]


@pytest.mark.parametrize("cdt", CDT)
@pytest.mark.parametrize("tr", TRANS)
def test_complex_brute_force_small(cdt, tr):
    for M, N, K in itertools.product(range(1, 5), repeat=3):
        c = CCase(cdt, tr[0], tr[1], M, N, K, 9, 40 + M, 0.5 - 1.25j, 1j, pad=1, spad=1)
        c.run()
        torch.cuda.synchronize()
        c.check()


@pytest.mark.parametrize("cdt", CDT)
@pytest.mark.parametrize("tr", TRANS)
def test_complex_square_sweep(cdt, tr):
    for n in (5, 8, 13, 16, 24, 32, 40, 56, 64, 80):
        if tr == "TN" and n > 32:
            continue
        if cdt == np.complex128 and n > 56 and n % 8:
            continue  # large ZGEMM runs on the K-streamed DMMA kernels (M, N multiples of 8)
        for alpha, beta in ((1.5 - 0.5j, 0.25 + 1j), (-1j, 0)):
            c = CCase(cdt, tr[0], tr[1], n, n, n, 1203, 7, alpha, beta)
            if beta == 0:
                c.C.fill_(float("nan"))  # beta == 0: C is write-only
            c.run()
            torch.cuda.synchronize()
            c.check(sample_ids(c.batch, 128, 64))


@pytest.mark.parametrize("cdt", CDT)
def test_complex_tn_extended_domain(cdt):
    """complex TN above 32^3 once the caller widens the TN bound."""
    from paper_2208_09822_b200 import iaat
    assert iaat.iaat_set_tn_limit(512000) == 0
    try:
        for (M, N, K) in ((40, 40, 40), (64, 64, 64), (80, 80, 80), (37, 53, 61)):
            if cdt == np.complex128 and (M % 8 or N % 8) and M * N * K > 175616:
                continue  # large ZGEMM runs on the K-streamed DMMA kernels (M, N multiples of 8)
            c = CCase(cdt, "T", "N", M, N, K, 301, 9, 1.5 - 0.5j, 0.25 + 1j)
            c.run()
            torch.cuda.synchronize()
            c.check(sample_ids(c.batch, 96, 32))
    finally:
        iaat.iaat_set_tn_limit(32768)


@pytest.mark.parametrize("cdt", CDT)
def test_complex_irregular_and_quick_returns(cdt):
    for (M, N, K) in ((7, 13, 5), (31, 3, 17), (1, 61, 9), (23, 23, 1)):
        c = CCase(cdt, "N", "T", M, N, K, 501, 3, 2 + 1j, -0.5j, pad=3)
        c.run()
        torch.cuda.synchronize()
        c.check(sample_ids(c.batch, 64, 32))
    # alpha = 0: C = beta*C, A/B never read (NaN-filled)
    c = CCase(cdt, "N", "N", 6, 5, 4, 33, 5, 0, 0.5 - 2j)
    c.A.fill_(float("nan"))
    c.B.fill_(float("nan"))
    c.run()
    torch.cuda.synchronize()
    c.check()
    # alpha = 0, beta = 1: no-op (C untouched)
    before = c.C.clone()
    c.alpha, c.beta = 0j, 1 + 0j
    c.run()
    torch.cuda.synchronize()
    assert torch.equal(before.view(torch.int64 if cdt == np.complex128 else torch.int32),
                       c.C.view(torch.int64 if cdt == np.complex128 else torch.int32))


@pytest.mark.parametrize("tr", TRANS)
def test_zgemm_k_streamed_dmma(tr):
    """ZGEMM on the fp64 tensor cores (K-streamed DMMA over the real view,
    forced family 3): every warp-tile size that divides the shape, ragged K
    chunks (K % 8 != 0: the copy engine's zero fill), a ragged last unit,
    complex alpha/beta with and without beta."""
    import os
    from paper_2208_09822_b200 import iaat
    shapes = [(64, 64, 64), (80, 80, 80), (16, 24, 37), (40, 32, 9), (8, 8, 8)]
    try:
        for (M, N, K) in shapes:
            if tr == "TN" and M * N * K > 32768:
                continue
            for wm in (1, 2, 4, 5):
                for wn in (1, 2, 3, 5):
                    if (M // 8) % wm or (N // 8) % wn:
                        continue
                    for beta, P in ((0j, 1), (0.5 - 0.25j, 2)):
                        os.environ["IAAT_FORCE_FAMILY"] = "3"
                        os.environ["IAAT_FORCE_TILE"] = "%dx%d" % (8 * wm, 8 * wn)
                        os.environ["IAAT_FORCE_P"] = str(P)
                        c = CCase(np.complex128, tr[0], tr[1], M, N, K, 97, 23, 1.25 + 0.5j, beta)
                        p = iaat.iaat_plan_describe(3, tr[0], tr[1], M, N, K, c.lda, c.sA, c.ldb, c.sB, c.ldc, c.sC,
                                                    c.batch, beta == 0)
                        if p.get("family") != "ks_dmma":
                            continue
                        if beta == 0:
                            c.C.fill_(float("nan"))
                        c.run()
                        torch.cuda.synchronize()
                        c.check(sample_ids(c.batch, 48, 24))
    finally:
        for k in ("IAAT_FORCE_FAMILY", "IAAT_FORCE_TILE", "IAAT_FORCE_P"):
            os.environ.pop(k, None)
