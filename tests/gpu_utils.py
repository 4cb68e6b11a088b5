"""Shared GPU-test machinery: seeded inputs on the device (datagen GPU twin),
the same inputs rebuilt on the host (datagen numpy) for the oracle, one call
through the C ABI, and the element-wise comparison of north_star:
    max |C_gpu - ref| / (|alpha| |opA||opB| + |beta| |C_in|)  <= tol.
"""
from __future__ import annotations

import numpy as np

import datagen
import oracle

TOL = {np.float32: 1e-5, np.float64: 1e-13}


def stored(trans, r_op, c_op):
    return (r_op, c_op) if trans == "N" else (c_op, r_op)


class Case:
    """One strided-batched problem set, resident on the GPU."""

    def __init__(self, dtype, tA, tB, M, N, K, batch, seed, alpha, beta, pad=0, spad=0,
                 first_id=0, elem_offset=0, ld_multiple=1):
        import torch
        self.dtype, self.tA, self.tB = dtype, tA, tB
        self.M, self.N, self.K, self.batch, self.seed = M, N, K, batch, seed
        self.alpha, self.beta = alpha, beta
        self.first_id = first_id
        ra, ca = stored(tA, M, K)
        rb, cb = stored(tB, K, N)
        self.ra, self.ca, self.rb, self.cb = ra, ca, rb, cb
        rup = lambda x: (x + ld_multiple - 1) // ld_multiple * ld_multiple  # noqa: E731
        self.lda, self.ldb, self.ldc = rup(max(1, ra) + pad), rup(max(1, rb) + pad), rup(max(1, M) + pad)
        self.sA = self.lda * ca + spad
        self.sB = self.ldb * cb + spad
        self.sC = self.ldc * N + spad
        tdt = torch.float32 if dtype == np.float32 else torch.float64
        self.off = elem_offset
        dev = "cuda"
        self.A = torch.empty(batch * self.sA + 16 + elem_offset, dtype=tdt, device=dev)
        self.B = torch.empty(batch * self.sB + 16 + elem_offset, dtype=tdt, device=dev)
        self.C = torch.empty(batch * self.sC + 16 + elem_offset, dtype=tdt, device=dev)
        for t in (self.A, self.B, self.C):
            t.fill_(float("nan"))
        o = elem_offset
        if batch and ra and ca:
            datagen.fill_device(self.A[o:], seed, datagen.MAT_A, ra, ca, self.lda, self.sA, batch, first_id)
        if batch and rb and cb:
            datagen.fill_device(self.B[o:], seed, datagen.MAT_B, rb, cb, self.ldb, self.sB, batch, first_id)
        if batch and M and N:
            datagen.fill_device(self.C[o:], seed, datagen.MAT_C, M, N, self.ldc, self.sC, batch, first_id)

    def views(self):
        o = self.off
        return self.A[o:], self.B[o:], self.C[o:]

    def run(self, check=True):
        from paper_2208_09822_b200 import iaat
        A, B, C = self.views()
        return iaat.gemm_strided_batched(self.tA, self.tB, self.M, self.N, self.K, self.alpha, A, self.lda,
                                         self.sA, B, self.ldb, self.sB, self.beta, C, self.ldc, self.sC,
                                         self.batch, check=check)

    def host_inputs(self, ids):
        """Rebuild the inputs of global problems `ids` on the host (packed)."""
        A = datagen.fill_host(self.seed, datagen.MAT_A, self.dtype, self.ra, self.ca, self.lda,
                              self.lda * self.ca, ids)
        B = datagen.fill_host(self.seed, datagen.MAT_B, self.dtype, self.rb, self.cb, self.ldb,
                              self.ldb * self.cb, ids)
        C = datagen.fill_host(self.seed, datagen.MAT_C, self.dtype, self.M, self.N, self.ldc,
                              self.ldc * self.N, ids)
        return A, B, C

    def oracle(self, local_ids):
        ids = np.asarray(local_ids, dtype=np.int64) + self.first_id
        A, B, C = self.host_inputs(ids)
        ref, den, _ = oracle.ref_gemm(self.tA, self.tB, self.M, self.N, self.K, self.alpha, A, self.lda,
                                      self.lda * self.ca, B, self.ldb, self.ldb * self.cb, self.beta, C,
                                      self.ldc, self.ldc * self.N, len(ids))
        return ref, den

    def gpu_result(self, local_ids):
        """C_gpu of the given local problems as (n, N, M) float64."""
        import torch
        C = self.views()[2]
        ids = torch.as_tensor(np.asarray(local_ids, dtype=np.int64), device=C.device)
        j = torch.arange(self.N, device=C.device).view(1, -1, 1) * self.ldc
        i = torch.arange(self.M, device=C.device).view(1, 1, -1)
        idx = ids.view(-1, 1, 1) * self.sC + j + i
        return C[idx].double().cpu().numpy()

    def check(self, local_ids=None, tol=None):
        if local_ids is None:
            local_ids = np.arange(self.batch)
        ref, den = self.oracle(local_ids)
        got = self.gpu_result(local_ids)
        err = oracle.max_rel_err(got, ref, den)
        tol = TOL[self.dtype] if tol is None else tol
        assert err <= tol, "max rel err %.3e > %.1e (%s%s M=%d N=%d K=%d)" % (
            err, tol, self.tA, self.tB, self.M, self.N, self.K)
        return err, got, ref


def sample_ids(batch, n_rand=1024, edge=256, seed=0):
    rng = np.random.default_rng(seed)
    ids = set(range(min(edge, batch)))
    ids |= set(range(max(0, batch - edge), batch))
    ids |= set(rng.integers(0, batch, size=min(n_rand, batch)).tolist())
    return np.array(sorted(ids), dtype=np.int64)


# BASELINE.json configs ------------------------------------------------------
S3 = [1, 3, 5, 7, 11, 13, 17, 23, 31, 37, 47, 53, 61, 67, 79]


def config3_shapes():
    """64 distinct (M,N,K) drawn without replacement from the sorted S^3
    with numpy.random.default_rng(2) (DESIGN.md input recipe, config 3)."""
    triples = [(m, n, k) for m in S3 for n in S3 for k in S3 if m * n * k <= 512000]
    rng = np.random.default_rng(2)
    pick = rng.choice(len(triples), size=64, replace=False)
    return [triples[i] for i in pick]


def config4_shapes():
    return [(n, n, n) for n in range(2, 33)] + [(32, 32, 2), (2, 32, 32)]


def config2_batch(n, elt=4):
    return (256 * 1024 * 1024) // ((3 * n * n) * elt)


# ---------------------------------------------------------------- complex
CTOL = {np.complex64: 1e-5, np.complex128: 1e-13}


class CCase:
    """One strided-batched complex problem set on the GPU.  Interleaved
    (re, im) data are generated as a real (2*rows) x cols matrix with real
    ld 2*ld by the same counter generator (no new generator arithmetic)."""

    def __init__(self, cdtype, tA, tB, M, N, K, batch, seed, alpha, beta, pad=0, spad=0):
        import torch
        self.cdtype, self.tA, self.tB = cdtype, tA, tB
        self.rdtype = np.float32 if cdtype == np.complex64 else np.float64
        self.M, self.N, self.K, self.batch, self.seed = M, N, K, batch, seed
        self.alpha, self.beta = complex(alpha), complex(beta)
        ra, ca = stored(tA, M, K)
        rb, cb = stored(tB, K, N)
        self.ra, self.ca, self.rb, self.cb = ra, ca, rb, cb
        self.lda, self.ldb, self.ldc = max(1, ra) + pad, max(1, rb) + pad, max(1, M) + pad
        self.sA, self.sB, self.sC = self.lda * ca + spad, self.ldb * cb + spad, self.ldc * N + spad
        tdt = torch.float32 if self.rdtype == np.float32 else torch.float64
        self.A = torch.full((2 * (batch * self.sA + 8),), float("nan"), dtype=tdt, device="cuda")
        self.B = torch.full((2 * (batch * self.sB + 8),), float("nan"), dtype=tdt, device="cuda")
        self.C = torch.full((2 * (batch * self.sC + 8),), float("nan"), dtype=tdt, device="cuda")
        if batch:
            datagen.fill_device(self.A, seed, datagen.MAT_A, 2 * ra, ca, 2 * self.lda, 2 * self.sA, batch)
            datagen.fill_device(self.B, seed, datagen.MAT_B, 2 * rb, cb, 2 * self.ldb, 2 * self.sB, batch)
            datagen.fill_device(self.C, seed, datagen.MAT_C, 2 * M, N, 2 * self.ldc, 2 * self.sC, batch)

    def run(self, check=True):
        from paper_2208_09822_b200 import iaat
        dt = iaat.IAAT_C32F if self.cdtype == np.complex64 else iaat.IAAT_C64F
        st = iaat.iaat_gemm_strided_batched(dt, self.tA, self.tB, self.M, self.N, self.K, self.alpha,
                                            self.A.data_ptr(), self.lda, self.sA, self.B.data_ptr(), self.ldb,
                                            self.sB, self.beta, self.C.data_ptr(), self.ldc, self.sC, self.batch)
        if check and st != 0:
            raise iaat.IaatError(st)
        return st

    def host(self, mat, rows, cols, ld, ids):
        re = datagen.fill_host(self.seed, mat, self.rdtype, 2 * rows, cols, 2 * ld, 2 * ld * cols, ids)
        return re.view(self.cdtype)

    def oracle(self, ids):
        ids = np.asarray(ids, dtype=np.int64)
        A = self.host(datagen.MAT_A, self.ra, self.ca, self.lda, ids)
        B = self.host(datagen.MAT_B, self.rb, self.cb, self.ldb, ids)
        C = self.host(datagen.MAT_C, self.M, self.N, self.ldc, ids)
        ref, den, _ = oracle.ref_cgemm(self.tA, self.tB, self.M, self.N, self.K, self.alpha, A, self.lda,
                                       self.lda * self.ca, B, self.ldb, self.ldb * self.cb, self.beta, C, self.ldc,
                                       self.ldc * self.N, len(ids))
        return ref, den

    def gpu_result(self, ids):
        import torch
        C = self.C.view(-1, 2)
        ids = torch.as_tensor(np.asarray(ids, dtype=np.int64), device=C.device)
        j = torch.arange(self.N, device=C.device).view(1, -1, 1) * self.ldc
        i = torch.arange(self.M, device=C.device).view(1, 1, -1)
        idx = ids.view(-1, 1, 1) * self.sC + j + i
        v = C[idx].double().cpu().numpy()
        return v[..., 0] + 1j * v[..., 1]

    def check(self, ids=None, tol=None):
        if ids is None:
            ids = np.arange(self.batch)
        ref, den = self.oracle(ids)
        got = self.gpu_result(ids)
        err = oracle.max_rel_err_complex(got, ref, den)
        tol = CTOL[self.cdtype] if tol is None else tol
        assert err <= tol, "complex max rel err %.3e > %.1e (%s%s M=%d N=%d K=%d)" % (
            err, tol, self.tA, self.tB, self.M, self.N, self.K)
        return err
