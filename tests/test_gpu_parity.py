"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Element-wise, on seeded inputs, within north_star's tolerances (1e-5 fp32,
1e-13 fp64, normalised by |alpha||opA||opB| + |beta||C|); bitwise where the
arithmetic is exact (integer-valued inputs, P4) or where the design fixes it
(determinism, batch-split invariance, fp32 transpose identity).
"""
from __future__ import annotations

import itertools

import numpy as np
import pytest

from tests.gpu_utils import Case, TOL, config2_batch, config3_shapes, config4_shapes, sample_ids

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2208_09822_b200 import iaat  # noqa: F401  (fails loudly if not built)
    yield


F32, F64 = np.float32, np.float64
TRANS = ["NN", "NT", "TN", "TT"]


def bits_equal(a, b):
    """Bitwise tensor equality (NaN payloads included)."""
    it = torch.int32 if a.dtype == torch.float32 else torch.int64
    return torch.equal(a.view(it), b.view(it))


# ---------------------------------------------------------------- datagen twin
def test_datagen_gpu_twin_bitwise():
    import datagen
    for dt, tdt in ((F32, torch.float32), (F64, torch.float64)):
        t = torch.empty(3 * 45, dtype=tdt, device="cuda")
        datagen.fill_device(t, 7, datagen.MAT_B, 5, 6, 7, 45, 3, first_id=11)
        want = datagen.fill_host(7, datagen.MAT_B, dt, 5, 6, 7, 45, [11, 12, 13])
        got = t.cpu().numpy()
        assert np.array_equal(np.isnan(got), np.isnan(want))
        m = ~np.isnan(want)
        assert np.array_equal(got[m].view(np.uint8), want[m].view(np.uint8))


# ---------------------------------------------------------------- brute force 1..4^3
@pytest.mark.parametrize("dtype", [F32, F64])
@pytest.mark.parametrize("tr", TRANS)
def test_brute_force_small(dtype, tr):
    """P8: every (M,N,K) in {1..4}^3, this transposition, several alpha/beta,
    minimal and padded ld (NaN sentinels in the padding and between problems)."""
    ab = [(1.0, 0.0), (1.5, 0.5), (-1.0, 1.0), (0.5, -1.0)]
    for (M, N, K), (alpha, beta), pad in itertools.product(itertools.product(range(1, 5), repeat=3), ab, (0, 3)):
        c = Case(dtype, tr[0], tr[1], M, N, K, 5, 100 + M * 16 + N * 4 + K, alpha, beta, pad=pad, spad=pad)
        c.run()
        c.check()


# ---------------------------------------------------------------- configs (reduced batch, every problem)
@pytest.mark.parametrize("tr", ["NN", "NT", "TT"])
def test_config2_square_sweep(tr):
    for n in range(4, 81, 4):
        c = Case(F32, tr[0], tr[1], n, n, n, 600, 1, 1.5, 0.5)
        c.run()
        c.check()


def test_config1_full():
    c = Case(F32, "N", "N", 16, 16, 16, 2000, 0, 1.0, 0.0)
    c.run()
    c.check()


def test_config3_irregular():
    for (M, N, K) in config3_shapes():
        c = Case(F32, "N", "N", M, N, K, 300, 2, 1.0, 1.0)
        c.run()
        c.check()


@pytest.mark.parametrize("tr", ["NT", "TT"])
def test_config3_irregular_other_trans(tr):
    for (M, N, K) in config3_shapes()[::4]:
        c = Case(F32, tr[0], tr[1], M, N, K, 200, 2, 1.0, 1.0)
        c.run()
        c.check()


def test_config4_tn():
    for (M, N, K) in config4_shapes():
        c = Case(F32, "T", "N", M, N, K, 1000, 3, -1.0, 0.25)
        c.run()
        c.check()


@pytest.mark.parametrize("tr", ["NN", "NT"])
def test_config5_fp64(tr):
    for n in (8, 16, 32, 48, 64, 80):
        c = Case(F64, tr[0], tr[1], n, n, n, 400, 4, 1.0, 0.0)
        c.run()
        c.check()


@pytest.mark.parametrize("tr", ["TN", "TT"])
def test_fp64_other_trans(tr):
    for (M, N, K) in [(8, 8, 8), (16, 24, 13), (31, 17, 23), (32, 32, 32)]:
        c = Case(F64, tr[0], tr[1], M, N, K, 300, 40, 1.5, -0.5)
        c.run()
        c.check()


def test_fp64_odd_shapes():
    for (M, N, K) in [(7, 9, 11), (23, 5, 41), (79, 79, 79), (1, 80, 80), (80, 1, 3), (13, 64, 7)]:
        for tr in TRANS:
            if tr == "TN" and M * N * K > 32768:
                continue
            c = Case(F64, tr[0], tr[1], M, N, K, 64, 41, 1.0, 1.0)
            c.run()
            c.check()


@pytest.mark.parametrize("dtype", [F32, F64])
def test_tn_extended_domain(dtype):
    """TN above 32^3 once the caller widens the TN bound."""
    from paper_2208_09822_b200 import iaat
    big = Case(dtype, "T", "N", 40, 40, 40, 8, 5, 1.0, 0.0)
    assert big.run(check=False) == 2  # IAAT_ERROR_NOT_SMALL by default
    assert iaat.iaat_set_tn_limit(512000) == 0
    try:
        for (M, N, K) in [(33, 33, 33), (48, 48, 48), (64, 64, 64), (80, 80, 80), (79, 79, 79),
                          (40, 72, 56), (1, 80, 80), (80, 3, 77), (68, 76, 52)]:
            c = Case(dtype, "T", "N", M, N, K, 300, 43, 1.5, -0.5)
            c.run()
            c.check()
    finally:
        iaat.iaat_set_tn_limit(32768)


# ---------------------------------------------------------------- full-size launch configs, sampled
@pytest.mark.parametrize("tr", ["NN", "NT", "TT"])
@pytest.mark.parametrize("n", list(range(4, 81, 4)))
def test_config2_full_batch_sampled(n, tr):
    """The bench's launch configuration (config 2 full batch, the plan the
    bench runs -- tuned table entry or cost model), checked on the first /
    last 256 problems and 1024 seeded random ones."""
    c = Case(F32, tr[0], tr[1], n, n, n, config2_batch(n), 1, 1.5, 0.5)
    c.run()
    c.check(sample_ids(c.batch))


@pytest.mark.parametrize("i", range(64))
def test_config3_full_batch_sampled(i):
    """Config 3 at its bench batch (100000 per shape), sampled."""
    M, N, K = config3_shapes()[i]
    c = Case(F32, "N", "N", M, N, K, 100000, 2, 1.0, 1.0)
    c.run()
    c.check(sample_ids(c.batch))


@pytest.mark.parametrize("shape", config4_shapes())
def test_config4_full_batch_sampled(shape):
    """Config 4 (TN) at its bench batch (500000 per shape), sampled."""
    M, N, K = shape
    c = Case(F32, "T", "N", M, N, K, 500000, 3, -1.0, 0.25)
    c.run()
    c.check(sample_ids(c.batch))


@pytest.mark.parametrize("tr", ["NN", "NT"])
@pytest.mark.parametrize("n", [32, 80])
def test_config5_full_batch_sampled(n, tr):
    """Config 5 (fp64) at the bench's launch size: the full 2e6 batch where
    it fits, else one bench chunk (60 % of HBM, bench.py)."""
    per = 3 * n * n * 8
    cap = int(0.60 * torch.cuda.get_device_properties(0).total_memory) // per
    c = Case(F64, tr[0], tr[1], n, n, n, min(2_000_000, cap), 4, 1.0, 0.0)
    c.run()
    c.check(sample_ids(c.batch))
    del c
    torch.cuda.empty_cache()


# ---------------------------------------------------------------- exactness / invariants
@pytest.mark.parametrize("dtype", [F32, F64])
@pytest.mark.parametrize("tr", TRANS)
def test_integer_inputs_bitwise(dtype, tr):
    """P4: integer entries -> every product and partial sum is exact, so the
    GPU equals the (exact) oracle bitwise for any summation order."""
    from paper_2208_09822_b200 import iaat
    rng = np.random.default_rng(44)
    M, N, K, batch = 13, 11, 30, 50
    ra, ca = (M, K) if tr[0] == "N" else (K, M)
    rb, cb = (K, N) if tr[1] == "N" else (N, K)
    A = rng.integers(-8, 9, batch * ra * ca).astype(dtype)
    B = rng.integers(-8, 9, batch * rb * cb).astype(dtype)
    C = rng.integers(-8, 9, batch * M * N).astype(dtype)
    import oracle
    ref, _, _ = oracle.ref_gemm(tr[0], tr[1], M, N, K, 0.5, A, ra, ra * ca, B, rb, rb * cb, -1.5, C, M, M * N, batch)
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
    iaat.gemm_strided_batched(tr[0], tr[1], M, N, K, 0.5, dA, ra, ra * ca, dB, rb, rb * cb, -1.5, dC, M, M * N, batch)
    got = dC.cpu().numpy().astype(np.float64).reshape(batch, N, M)
    assert np.array_equal(got, ref)


def test_dependent_calls_in_stream_order():
    """Back-to-back calls on one stream where each reads the previous call's
    C (programmatic dependent launch: the next grid may launch early but must
    wait for its predecessor before reading).  Integer inputs keep every
    value exact, so the chain is compared bitwise with int64 numpy; the
    shapes alternate between the slab and the K-streamed families."""
    from paper_2208_09822_b200 import iaat
    rng = np.random.default_rng(45)
    batch, n = 3000, 48
    # entries in {-1, 0, 1}: after 4 products |value| <= 48^4 < 2^24, exact in fp32
    A = rng.integers(-1, 2, (batch, n, n)).astype(np.float32)  # stored column-major: [b][col][row]
    B = rng.integers(-1, 2, (batch, n, n)).astype(np.float32)
    dX = torch.from_numpy(A).cuda().reshape(-1)
    dB = torch.from_numpy(B).cuda().reshape(-1)
    outs = [torch.empty_like(dX) for _ in range(4)]
    ref = A.astype(np.int64)
    Bi = B.astype(np.int64)
    src = dX
    for step, out in enumerate(outs):
        # C_col[b] = X_col[b] @ B_col[b]; in [b][col][row] storage that is (B^T X^T)^T
        _force(**({"family": 2} if step % 2 else {}))
        try:
            iaat.gemm_strided_batched("N", "N", n, n, n, 1.0, src, n, n * n, dB, n, n * n, 0.0, out, n, n * n, batch)
        finally:
            _force()
        ref = np.einsum("bkr,bck->bcr", ref, Bi)  # X[b][k][r] * B[b][c][k] -> C[b][c][r]
        src = out
    torch.cuda.synchronize()
    assert np.abs(ref).max() < 2 ** 24  # exact in fp32 all along
    got = outs[-1].cpu().numpy().astype(np.int64).reshape(batch, n, n)
    assert np.array_equal(got, ref)


def test_single_process_device_loop_matches_one_call():
    """dist.gemm_on_devices: shards of one batch issued per device from one
    process (here every shard on cuda:0, the only GPU) equal one
    unsharded call bitwise."""
    from paper_2208_09822_b200 import dist
    n, batch = 40, 1001
    one = Case(F32, "N", "T", n, n, n, batch, 61, 1.5, 0.5)
    parts = Case(F32, "N", "T", n, n, n, batch, 61, 1.5, 0.5)
    one.run()
    A, B, C = parts.views()
    calls = []
    for g in range(3):
        lo, hi = dist.shard_range(batch, g, 3)
        calls.append((0, dict(transA="N", transB="T", M=n, N=n, K=n, alpha=1.5, A=A[lo * parts.sA:], lda=parts.lda,
                              strideA=parts.sA, B=B[lo * parts.sB:], ldb=parts.ldb, strideB=parts.sB, beta=0.5,
                              C=C[lo * parts.sC:], ldc=parts.ldc, strideC=parts.sC, batch=hi - lo)))
    dist.gemm_on_devices(calls)
    torch.cuda.synchronize()
    assert bits_equal(one.views()[2][:batch * one.sC], C[:batch * parts.sC])


def test_transpose_identity_fp32_bitwise():
    """P7: op(A)op(B) = (op(B)^T op(A)^T)^T -- one k-ascending FFMA chain per
    element and fma(a,b,c) = fma(b,a,c) make the two calls bitwise equal."""
    from paper_2208_09822_b200 import iaat
    flip = {"N": "T", "T": "N"}
    for tr in TRANS:
        M, N, K, batch = 19, 12, 37, 40
        c1 = Case(F32, tr[0], tr[1], M, N, K, batch, 77, 1.0, 0.0)
        c1.run()
        A, B, _ = c1.views()
        C2 = torch.empty(batch * N * M, dtype=torch.float32, device="cuda")
        iaat.gemm_strided_batched(flip[tr[1]], flip[tr[0]], N, M, K, 1.0, B, c1.ldb, c1.sB, A, c1.lda, c1.sA,
                                  0.0, C2, N, N * M, batch)
        g1 = c1.gpu_result(np.arange(batch))
        # C2 is N x M column-major (ldc = N): C2[b][i*N + j] = C2(j, i) = C(i, j)
        g2 = C2.view(batch, M, N).double().cpu().numpy().transpose(0, 2, 1)
        assert np.array_equal(g1, g2), tr


def test_determinism_and_batch_split_invariance():
    """P11: two runs and a 3-way split of the batch give bitwise equal C."""
    from paper_2208_09822_b200 import iaat
    for dtype, n in ((F32, 24), (F64, 32)):
        c = Case(dtype, "N", "T", n, n, n, 3001, 9, 1.0, 0.0)
        c.run()
        r1 = c.views()[2].clone()
        c.run()
        assert bits_equal(r1, c.views()[2])
        A, B, C = c.views()
        C.fill_(float("nan"))
        cuts = [0, 1000, 1777, 3001]
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            iaat.gemm_strided_batched("N", "T", n, n, n, 1.0, A[lo * c.sA:], c.lda, c.sA, B[lo * c.sB:], c.ldb,
                                      c.sB, 0.0, C[lo * c.sC:], c.ldc, c.sC, hi - lo)
        assert bits_equal(r1, C)


def test_beta_zero_ignores_nan_c_and_alpha_zero_ignores_ab():
    from paper_2208_09822_b200 import iaat
    c = Case(F32, "N", "N", 9, 7, 5, 100, 5, 1.0, 0.0)
    c.views()[2].fill_(float("nan"))
    c.run()
    assert np.isfinite(c.gpu_result(np.arange(100))).all()
    c.check()
    # alpha = 0: A and B are never read (NaN), C = beta*C
    c2 = Case(F64, "T", "T", 9, 7, 5, 100, 6, 0.0, 2.0)
    c2.views()[0].fill_(float("nan"))
    c2.views()[1].fill_(float("nan"))
    c2.run()
    c2.check()
    # alpha = 0, beta = 0: zeros without reading C
    c3 = Case(F32, "N", "N", 9, 7, 5, 100, 6, 0.0, 0.0)
    c3.views()[2].fill_(float("nan"))
    A, B, C = c3.views()
    iaat.gemm_strided_batched("N", "N", 9, 7, 5, 0.0, A, c3.lda, c3.sA, B, c3.ldb, c3.sB, 0.0, C, c3.ldc, c3.sC, 100)
    assert (torch.from_numpy(c3.gpu_result(np.arange(100))) == 0).all()
    # K = 0: C = beta * C
    c4 = Case(F32, "N", "N", 9, 7, 0, 50, 8, 1.0, 0.5)
    c4.run()
    c4.check()


def test_quick_returns_leave_c_untouched():
    from paper_2208_09822_b200 import iaat
    c = Case(F32, "N", "N", 8, 8, 8, 10, 5, 0.0, 1.0)
    before = c.views()[2].clone()
    n0 = iaat.iaat_launch_count()
    c.run()  # alpha = 0, beta = 1: no-op, nothing enqueued
    assert iaat.iaat_launch_count() == n0
    assert bits_equal(before, c.views()[2])
    A, B, C = c.views()
    for M, N, batch in ((0, 8, 10), (8, 0, 10), (8, 8, 0)):
        st = iaat.gemm_strided_batched("N", "N", M, N, 8, 1.0, A, 8, 64, B, 8, 64, 0.0, C, 8, 64, batch)
        assert st == 0
    assert bits_equal(before, c.views()[2])


def test_misaligned_bases_and_padding():
    """Base pointers one element off 16 B, ld padding and problem gaps (NaN
    sentinels that must never be read), a canary after the last C."""
    for dtype in (F32, F64):
        for tr in TRANS:
            M, N, K = (13, 7, 11) if tr != "TN" else (9, 9, 9)
            c = Case(dtype, tr[0], tr[1], M, N, K, 333, 12, 1.25, -0.75, pad=3, spad=5, elem_offset=1)
            C = c.views()[2]
            tail = C[333 * c.sC:].clone()
            c.run()
            c.check()
            assert bits_equal(tail, C[333 * c.sC:])


def test_padding_between_columns_untouched():
    c = Case(F32, "N", "N", 10, 6, 7, 77, 13, 1.0, 0.0, pad=4)
    c.run()
    C = c.views()[2].cpu().numpy()
    for b in range(77):
        for j in range(6):
            s = b * c.sC + j * c.ldc
            assert np.all(np.isnan(C[s + 10:s + 14]))


def test_broadcast_stride_zero():
    """strideA = 0: every problem uses the same A."""
    from paper_2208_09822_b200 import iaat
    import datagen
    import oracle
    M, N, K, batch = 12, 20, 16, 500
    A = datagen.fill_host(21, 0, F32, M, K, M, M * K, [0])
    B = datagen.fill_host(21, 1, F32, K, N, K, K * N, list(range(batch)))
    ref, den, _ = oracle.ref_gemm("N", "N", M, N, K, 1.0, A, M, 0, B, K, K * N, 0.0, None, M, M * N, batch)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC = torch.empty(batch * M * N, dtype=torch.float32, device="cuda")
    iaat.gemm_strided_batched("N", "N", M, N, K, 1.0, dA, M, 0, dB, K, K * N, 0.0, dC, M, M * N, batch)
    got = dC.view(batch, N, M).double().cpu().numpy()
    assert oracle.max_rel_err(got, ref, den) <= 1e-5


# ---------------------------------------------------------------- pointer-array API
@pytest.mark.parametrize("dtype", [F32, F64])
def test_pointer_array_api_shuffled_and_aliased(dtype):
    from paper_2208_09822_b200 import iaat
    import oracle
    rng = np.random.default_rng(3)
    for tr, (M, N, K) in (("NN", (16, 16, 16)), ("TN", (7, 9, 5)), ("NT", (33, 17, 29)), ("TT", (8, 24, 40))):
        batch = 257
        c = Case(dtype, tr[0], tr[1], M, N, K, batch, 31, 1.5, 0.5)
        A, B, C = c.views()
        perm = rng.permutation(batch)  # problem b of the call uses storage slot perm[b]
        esz = A.element_size()
        Ap = torch.tensor([A.data_ptr() + int(s) * c.sA * esz for s in perm], dtype=torch.int64, device="cuda")
        Bp = torch.tensor([B.data_ptr() + int(s) * c.sB * esz for s in perm], dtype=torch.int64, device="cuda")
        Cp = torch.tensor([C.data_ptr() + int(s) * c.sC * esz for s in perm], dtype=torch.int64, device="cuda")
        iaat.gemm_batched(tr[0], tr[1], M, N, K, 1.5, Ap, c.lda, Bp, c.ldb, 0.5, Cp, c.ldc, batch,
                          dtype=0 if dtype == F32 else 1)
        c.check()  # slot s holds problem s's inputs and must hold its result
    # aliased A and B (same storage): C = A * A^T
    M = K = 12
    N = 12
    c = Case(dtype, "N", "T", M, N, K, 64, 32, 1.0, 0.0)
    A = c.views()[0]
    esz = A.element_size()
    Ap = torch.tensor([A.data_ptr() + b * c.sA * esz for b in range(64)], dtype=torch.int64, device="cuda")
    C = c.views()[2]
    Cp = torch.tensor([C.data_ptr() + b * c.sC * esz for b in range(64)], dtype=torch.int64, device="cuda")
    iaat.gemm_batched("N", "T", M, N, K, 1.0, Ap, c.lda, Ap, c.lda, 0.0, Cp, c.ldc, 64,
                      dtype=0 if dtype == F32 else 1)
    Ah = A[:64 * c.sA].double().cpu().numpy()
    ref, den, _ = oracle.ref_gemm("N", "T", M, N, K, 1.0, Ah, c.lda, c.sA, Ah, c.lda, c.sA, 0.0, None, c.ldc,
                                  c.sC, 64)
    got = c.gpu_result(np.arange(64))
    assert oracle.max_rel_err(got, ref, den) <= TOL[dtype]


# ---------------------------------------------------------------- error statuses
def test_invalid_arguments_enqueue_nothing():
    from paper_2208_09822_b200 import iaat
    c = Case(F32, "N", "N", 8, 8, 8, 4, 1, 1.0, 0.0)
    A, B, C = c.views()
    before = C.clone()
    n0 = iaat.iaat_launch_count()
    f = iaat.iaat_gemm_strided_batched
    a, b, cc = A.data_ptr(), B.data_ptr(), C.data_ptr()
    assert f(0, "C", "N", 8, 8, 8, 1.0, a, 8, 64, b, 8, 64, 0.0, cc, 8, 64, 4) == 1
    assert f(0, "N", "N", -1, 8, 8, 1.0, a, 8, 64, b, 8, 64, 0.0, cc, 8, 64, 4) == 1
    assert f(0, "N", "N", 8, 8, 8, 1.0, a, 7, 64, b, 8, 64, 0.0, cc, 8, 64, 4) == 1   # lda < M
    assert f(0, "N", "N", 8, 8, 8, 1.0, a, 8, 64, b, 8, 64, 0.0, cc, 8, 10, 4) == 1   # overlapping C
    assert f(0, "N", "N", 8, 8, 8, 1.0, a + 2, 8, 64, b, 8, 64, 0.0, cc, 8, 64, 4) == 1  # misaligned
    assert f(0, "N", "N", 8, 8, 8, 1.0, 0, 8, 64, b, 8, 64, 0.0, cc, 8, 64, 4) == 1   # NULL A
    assert f(0, "N", "N", 81, 81, 81, 1.0, a, 81, 64, b, 81, 64, 0.0, cc, 81, 6561, 4) == 2
    assert f(0, "T", "N", 33, 33, 33, 1.0, a, 33, 64, b, 33, 64, 0.0, cc, 33, 1089, 4) == 2
    assert f(7, "N", "N", 8, 8, 8, 1.0, a, 8, 64, b, 8, 64, 0.0, cc, 8, 64, 4) == 1
    torch.cuda.synchronize()
    assert iaat.iaat_launch_count() == n0
    assert bits_equal(before, C)


def test_launch_uses_sm100_kernels_only():
    """The call enqueues exactly one launch (the persistent plan), and the
    kernels the device actually ran (CUDA activity trace) are this library's
    own iaat_* kernels -- no library or fallback kernel -- for every family
    (slab, K-streamed, ksg, fp64 DMMA); the shipped .so holds sm_100a SASS
    only (tests/test_build.py)."""
    import os
    from torch.profiler import ProfilerActivity, profile
    from paper_2208_09822_b200 import iaat
    c = Case(F32, "N", "N", 32, 32, 32, 1000, 1, 1.0, 0.0)
    n0 = iaat.iaat_launch_count()
    c.run()
    assert iaat.iaat_launch_count() == n0 + 1
    torch.cuda.synchronize()
    cases = [Case(F32, "N", "N", 16, 16, 16, 500, 1, 1.0, 0.0), Case(F32, "N", "T", 64, 64, 64, 300, 2, 1.5, 0.5),
             Case(F64, "N", "N", 32, 32, 32, 300, 3, 1.0, 0.0), Case(F32, "T", "T", 40, 36, 44, 129, 4, 1.5, 0.5)]
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i, cc in enumerate(cases):
            if i == 3:
                os.environ["IAAT_FORCE_FAMILY"] = "2"
            try:
                cc.run()
            finally:
                os.environ.pop("IAAT_FORCE_FAMILY", None)
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
    kern = [n for n in names if "memcpy" not in n.lower() and "memset" not in n.lower()]
    assert len([n for n in kern if "iaat" in n]) == len(cases), kern
    assert all("iaat" in n for n in kern), kern
    assert any("iaat_ksg_" in n for n in kern) and any("iaat_ks_" in n or "iaat_ks1_" in n for n in kern), kern


# ---------------------------------------------------------------- K-streamed (TMA) family
KS_SHAPES = [(64, 64, 64), (80, 80, 80), (36, 44, 52), (20, 28, 12), (8, 8, 8), (48, 40, 37), (76, 68, 96)]


def _force(**kw):
    import os
    for k in ("IAAT_FORCE_FAMILY", "IAAT_FORCE_TILE", "IAAT_FORCE_P", "IAAT_FORCE_CTAS", "IAAT_FORCE_ORDER",
              "IAAT_FORCE_S"):
        os.environ.pop(k, None)
    for k, v in kw.items():
        os.environ["IAAT_FORCE_" + k.upper()] = str(v)


@pytest.mark.parametrize("tr", TRANS)
@pytest.mark.parametrize("dtype", [F32, F64])
def test_ks_family_parity_and_bitwise_vs_slab(dtype, tr):
    """The K-streamed TMA plans (forced) against the oracle, on shapes with
    several tiles, ragged K chunks (K % 32, K % 4 != 0 with 16-byte padded
    ld), multi-class decompositions and a ragged last unit (batch % P); and
    fp32 bitwise equal to the slab family (same k-ascending FMA chain per
    element, same fused epilogue)."""
    from paper_2208_09822_b200 import iaat
    try:
        for (M, N, K) in KS_SHAPES:
            if tr == "TN" and M * N * K > 32768:
                continue
            for P, beta in ((1, 0.5), (3, 0.0)):
                if P > 1 and M * N > 2048:
                    continue  # P problems per unit must fit one CTA's warps
                _force(family=2, p=P)
                c = Case(dtype, tr[0], tr[1], M, N, K, 301, 21, 1.5, beta, ld_multiple=4)
                A, B, C = c.views()
                p = iaat.iaat_plan_describe(0 if dtype == F32 else 1, tr[0], tr[1], M, N, K, c.lda, c.sA, c.ldb,
                                            c.sB, c.ldc, c.sC, c.batch, beta == 0)
                assert p["family"].startswith("ks"), (tr, M, N, K, p["family"])
                c.run()
                torch.cuda.synchronize()
                c.check(sample_ids(c.batch, 64, 32))
                if dtype == F32:
                    ks = C.clone()
                    _force()
                    os_env_default = iaat.iaat_plan_describe(0, tr[0], tr[1], M, N, K, c.lda, c.sA, c.ldb, c.sB,
                                                             c.ldc, c.sC, c.batch, beta == 0)
                    c2 = Case(dtype, tr[0], tr[1], M, N, K, 301, 21, 1.5, beta, ld_multiple=4)
                    _force(family=0)
                    c2.run()
                    torch.cuda.synchronize()
                    assert bits_equal(ks, c2.views()[2]), (tr, M, N, K, os_env_default["family"])
    finally:
        _force()


@pytest.mark.parametrize("tr", TRANS)
@pytest.mark.parametrize("dtype", [F32, F64])
def test_ks_ldgsts_misaligned(dtype, tr):
    """Odd ld's / misaligned bases break the TMA 16-byte rules: the
    K-streamed plans then fill the same stages with cp.async (LDGSTS mode).
    Against the oracle on odd shapes (ragged chunks, ragged last unit,
    misaligned base, padded ld with NaN), and fp32 bitwise equal to the slab
    family."""
    from paper_2208_09822_b200 import iaat
    shapes = [(37, 41, 43), (7, 13, 5), (29, 29, 29), (61, 11, 79), (1, 31, 67)]
    try:
        for (M, N, K) in shapes:
            if tr == "TN" and M * N * K > 32768:
                continue
            for P, pad, off in ((1, 0, 0), (2, 1, 1)):
                _force(family=2, p=P)
                c = Case(dtype, tr[0], tr[1], M, N, K, 211, 17, -0.75, 1.25, pad=pad, elem_offset=off)
                p = iaat.iaat_plan_describe(0 if dtype == F32 else 1, tr[0], tr[1], M, N, K, c.lda, c.sA, c.ldb,
                                            c.sB, c.ldc, c.sC, c.batch, False, False, 256 if off == 0 else 4)
                if not p["family"].startswith("ks"):
                    continue  # e.g. P problems do not fit one CTA
                assert p["ldgsts"] == 1, (tr, M, N, K, p)
                c.run()
                torch.cuda.synchronize()
                c.check()
                if dtype == F32:
                    _force(family=0)
                    c2 = Case(dtype, tr[0], tr[1], M, N, K, 211, 17, -0.75, 1.25, pad=pad, elem_offset=off)
                    c2.run()
                    torch.cuda.synchronize()
                    assert bits_equal(c.views()[2], c2.views()[2]), (tr, M, N, K)
    finally:
        _force()


@pytest.mark.parametrize("tr", TRANS)
def test_ks_dmma_fp64_parity(tr):
    """fp64 K-streamed DMMA warp tiles (forced family 3) against the oracle:
    every warp-tile size that divides the shape, ragged K chunks (K % 16,
    K % 4 != 0 -> the copy engine's zero fill feeds the last DMMA step),
    a ragged last unit, beta = 0 and beta != 0."""
    from paper_2208_09822_b200 import iaat
    shapes = [(64, 64, 64), (80, 80, 80), (48, 32, 40), (16, 24, 37), (8, 8, 8), (56, 56, 56), (56, 16, 21)]
    try:
        for (M, N, K) in shapes:
            if tr == "TN" and M * N * K > 32768:
                continue
            for wm in (1, 2, 4, 5, 7):
                for wn in (1, 2, 3, 5, 7):
                    if (M // 8) % wm or (N // 8) % wn:
                        continue
                    for beta, P in ((0.0, 1), (0.5, 2)):
                        _force(family=3, tile="%dx%d" % (8 * wm, 8 * wn), p=P)
                        c = Case(F64, tr[0], tr[1], M, N, K, 203, 31, -1.25, beta, ld_multiple=2)
                        p = iaat.iaat_plan_describe(1, tr[0], tr[1], M, N, K, c.lda, c.sA, c.ldb, c.sB, c.ldc, c.sC,
                                                    c.batch, beta == 0)
                        if p["family"] != "ks_dmma":
                            continue  # (P x tiles) does not fit one CTA
                        c.run()
                        torch.cuda.synchronize()
                        c.check(sample_ids(c.batch, 48, 24))
    finally:
        _force()


@pytest.mark.parametrize("dtype", [F32, F64])
def test_grouped_variable_size_batches(dtype):
    """one grouped call over groups of different shapes,
    transpositions, alpha/beta and batch sizes equals the oracle, and is
    bitwise equal to the same groups called one by one."""
    from paper_2208_09822_b200 import iaat
    specs = [("N", "N", 7, 13, 5, 300, 1.0, 0.0), ("T", "N", 17, 3, 23, 1000, -1.0, 0.25),
             ("N", "T", 32, 32, 32, 500, 1.5, 0.5), ("T", "T", 1, 61, 7, 77, 2.0, 1.0),
             ("N", "N", 64, 48, 40, 200, 0.5, -0.5)]
    cases = [Case(dtype, ta, tb, M, N, K, b, 11 + i, al, be) for i, (ta, tb, M, N, K, b, al, be) in enumerate(specs)]
    ref_C = []
    for c in cases:  # group by group through the strided API
        c2 = Case(dtype, c.tA, c.tB, c.M, c.N, c.K, c.batch, c.seed, c.alpha, c.beta)
        c2.run()
        ref_C.append(c2)
    groups = []
    for c in cases:
        A, B, C = c.views()
        groups.append(dict(transA=c.tA, transB=c.tB, M=c.M, N=c.N, K=c.K, alpha=c.alpha, A=A.data_ptr(), lda=c.lda,
                           strideA=c.sA, B=B.data_ptr(), ldb=c.ldb, strideB=c.sB, beta=c.beta, C=C.data_ptr(),
                           ldc=c.ldc, strideC=c.sC, batch=c.batch))
    st = iaat.iaat_gemm_grouped_strided(0 if dtype == F32 else 1, groups,
                                        torch.cuda.current_stream().cuda_stream)
    assert st == 0
    torch.cuda.synchronize()
    for c, r in zip(cases, ref_C):
        c.check()
        assert bits_equal(c.views()[2], r.views()[2])


def test_grouped_argument_errors_enqueue_nothing():
    """Every group is validated and planned before any is enqueued: a NULL A
    or a misaligned base in the LAST group fails the call and leaves the C of
    every earlier group untouched (include/iaat.h, grouped API)."""
    from paper_2208_09822_b200 import iaat
    cases = [Case(F32, "N", "N", 16, 16, 16, 200, 3, 1.0, 0.5), Case(F32, "N", "T", 40, 40, 40, 100, 4, 1.0, 0.5),
             Case(F32, "T", "T", 9, 7, 5, 50, 5, 1.0, 0.5)]
    before = [c.views()[2].clone() for c in cases]

    def groups(bad):
        gs = []
        for i, c in enumerate(cases):
            A, B, C = c.views()
            a_ptr = A.data_ptr()
            if i == len(cases) - 1 and bad == "null":
                a_ptr = 0
            if i == len(cases) - 1 and bad == "misaligned":
                a_ptr += 2  # not element-aligned
            gs.append(dict(transA=c.tA, transB=c.tB, M=c.M, N=c.N, K=c.K, alpha=c.alpha, A=a_ptr, lda=c.lda,
                           strideA=c.sA, B=B.data_ptr(), ldb=c.ldb, strideB=c.sB, beta=c.beta, C=C.data_ptr(),
                           ldc=c.ldc, strideC=c.sC, batch=c.batch))
        return gs

    for bad in ("null", "misaligned"):
        st = iaat.iaat_gemm_grouped_strided(0, groups(bad), torch.cuda.current_stream().cuda_stream)
        assert st == 1, (bad, st)  # IAAT_ERROR_INVALID_VALUE
        torch.cuda.synchronize()
        for c, b0 in zip(cases, before):
            assert bits_equal(c.views()[2], b0), bad


@pytest.mark.parametrize("dtype", [F32, F64])
@pytest.mark.parametrize("tr", TRANS)
def test_elongated_in_domain_shapes(dtype, tr):
    """Shapes inside the small-GEMM domain whose single problem does not fit
    the slab family's shared memory (16 x 16 x 2000, 8 x 8 x 8000): the
    planner streams them through the K-streamed families instead of failing."""
    for (M, N, K) in ((16, 16, 2000), (8, 8, 8000), (80, 4, 1600)):
        if tr == "TN" and M * N * K > 32768:
            continue
        c = Case(dtype, tr[0], tr[1], M, N, K, 300, 9, 1.0, 0.5)
        c.run()
        torch.cuda.synchronize()
        c.check(sample_ids(c.batch, 64, 32))


@pytest.mark.parametrize("tr", ["NN", "NT"])
@pytest.mark.parametrize("n", [16, 64, 80])
def test_config5_shards_bitwise_equal_unsharded(n, tr):
    """Row e: config 5's strong-scaling shards -- each "rank" r
    of G generates its own inputs by GLOBAL problem id over
    dist.shard_range(B, r, G) and calls the library on them -- give C
    bitwise equal to one unsharded call, for G = 2, 4, 8 (shard boundaries
    included: every problem is compared)."""
    from paper_2208_09822_b200.dist import shard_range
    B = 20011
    full = Case(F64, tr[0], tr[1], n, n, n, B, 4, 1.0, 0.0)
    full.run()
    ref = full.views()[2].clone()
    del full
    for G in (2, 4, 8):
        parts = []
        for r in range(G):
            lo, hi = shard_range(B, r, G)
            c = Case(F64, tr[0], tr[1], n, n, n, hi - lo, 4, 1.0, 0.0, first_id=lo)
            c.run()
            parts.append(c.views()[2][:(hi - lo) * c.sC].clone())
        torch.cuda.synchronize()
        assert bits_equal(torch.cat(parts), ref[:B * n * n]), G
