/*
 * iaat.h -- C ABI of the B200-native batched small-GEMM library (libiaat.so).
 *
 * Operation (Sec. I): "GEMM is used to compute
 *     C = alpha A x B + beta C.  Here C, A, B are M x N, M x K and K x N".
 * with op(A), op(B) in {X, X^T}: "NT means matrix A is not transposed and
 * matrix B is transposed ... We acquiescence the matrix in column-major
 * order" (Table I note).  Small GEMM: cbrt(MNK) <= 80, or <= 32
 * when the transposition is TN (Sec. I), tested as the integer
 * M*N*K <= 512000 (32768 for TN) -- DESIGN.md reading A10.  The library runs
 * LARGE BATCHES of independent small problems, one problem per (A_b, B_b, C_b).
 *
 * Conventions (all entry points):
 *  - Column-major.  All sizes, leading dimensions and strides are int64_t
 *    counts of ELEMENTS.  Stored shapes (reading A1, BLAS):
 *      transA = 'N': A is M x K, lda >= max(1, M);  'T': A is K x M, lda >= max(1, K)
 *      transB = 'N': B is K x N, ldb >= max(1, K);  'T': B is N x K, ldb >= max(1, N)
 *      C is M x N, ldc >= max(1, M).
 *    transA/transB are the characters 'N','n','T','t' (anything else,
 *    including 'C', is IAAT_ERROR_INVALID_VALUE: transposition only).
 *  - alpha and beta are HOST pointers to one scalar of the call's dtype
 *    (float for IAAT_R32F, double for IAAT_R64F), or to two (re, im) for
 *    IAAT_C32F (float[2]) / IAAT_C64F (double[2]).
 *  - A, B, C (and the pointer arrays of iaat_gemm_batched together with the
 *    matrices they point to) are DEVICE memory of the current CUDA device.
 *    The caller owns every buffer; the library keeps only a host-side plan
 *    cache (thread-safe) and never allocates device memory on the call path.
 *  - Execution is asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *    default stream).  The call returns after enqueueing; buffers must stay
 *    alive until the stream's work completes.  Device faults surface at the
 *    caller's next synchronisation, as for any CUDA launch.  Kernels are
 *    launched with programmatic stream serialisation: a call's grid may
 *    start its prologue while the previous kernel on the stream drains, but
 *    it touches no global memory before that kernel has completed
 *    (griddepcontrol.wait), so stream order is preserved exactly.  Set
 *    IAAT_NO_PDL=1 in the environment to launch without it.
 *  - Validation happens before any launch.  On any error nothing is enqueued
 *    and C is untouched.  There is no CPU fallback: out-of-domain shapes
 *    return IAAT_ERROR_NOT_SMALL.
 *  - Quick returns (netlib/BLAS convention, readings A3-A5):
 *    M == 0, N == 0 or batch == 0: success, nothing enqueued.
 *    (alpha == 0 or K == 0) and beta == 1: success, nothing enqueued.
 *    alpha == 0 or K == 0 otherwise: C = beta*C (beta == 0 writes zeros and
 *    never reads C); A and B are never read.
 *    beta == 0: C is write-only (NaN/Inf in C never propagate).
 *  - Arithmetic: fp32 on CUDA-core FFMA (IEEE round-to-nearest, no TF32, no
 *    FTZ), fp64 on the DMMA tensor-core path / DFMA.  Each C element is one
 *    k-ascending FMA chain, so results do not depend on the plan, the batch
 *    split or the number of GPUs (bitwise deterministic).
 *  - Any element-aligned address is accepted; the planner chooses vector /
 *    bulk-copy paths from the actual alignment.
 */
#ifndef IAAT_H
#define IAAT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Data types.  Complex (the paper's CGEMM / ZGEMM rows, PAPER.md:
 * 96-97 Table I, Eq. 2): interleaved (re, im) element pairs,
 * every ld / stride counts COMPLEX elements, alpha / beta point to two
 * scalars (re, im); op is transposition only (N / T, no conjugation). */
typedef enum { IAAT_R32F = 0, IAAT_R64F = 1, IAAT_C32F = 2, IAAT_C64F = 3 } iaat_dtype_t;

typedef enum {
    IAAT_SUCCESS = 0,
    /* bad enum/char, negative size, ld < stored rows, stride < 0, C problems
       overlapping (strideC < (N-1)*ldc + M with batch > 1), NULL pointer where
       data must be read or written, pointer not element-aligned           */
    IAAT_ERROR_INVALID_VALUE = 1,
    /* M*N*K > 80^3 (> 32^3 for transA='T', transB='N') -- PAPER.md:36      */
    IAAT_ERROR_NOT_SMALL = 2,
    /* the current device is not compute capability 10.0 (sm_100a)         */
    IAAT_ERROR_ARCH = 3,
    /* a CUDA runtime call or the launch failed: see iaat_last_cuda_error()  */
    IAAT_ERROR_CUDA = 4,
    /* in-domain call the current kernels cannot stage (one problem's operand
       span exceeds shared memory, e.g. huge ld); nothing is enqueued        */
    IAAT_ERROR_NOT_SUPPORTED = 5
} iaat_status_t;

/* Strided batch: problem b uses A + b*strideA, B + b*strideB, C + b*strideC
 * (element offsets; strideA/strideB may be 0 to broadcast one matrix).     */
iaat_status_t iaat_gemm_strided_batched(
    iaat_dtype_t dtype, char transA, char transB, int64_t M, int64_t N, int64_t K,
    const void *alpha, const void *A, int64_t lda, int64_t strideA,
    const void *B, int64_t ldb, int64_t strideB,
    const void *beta, void *C, int64_t ldc, int64_t strideC,
    int64_t batch, void *stream);

/* Pointer-array batch (cuBLAS style): Aarray, Barray, Carray are DEVICE
 * arrays of `batch` DEVICE pointers.  C pointers of different problems must
 * not overlap (undefined behaviour otherwise, not checked).               */
iaat_status_t iaat_gemm_batched(
    iaat_dtype_t dtype, char transA, char transB, int64_t M, int64_t N, int64_t K,
    const void *alpha, const void *const *Aarray, int64_t lda,
    const void *const *Barray, int64_t ldb,
    const void *beta, void *const *Carray, int64_t ldc,
    int64_t batch, void *stream);

/* Grouped (variable-size) strided batches: group g is one
 * strided batched call with its own transA[g], transB[g], M[g], N[g], K[g],
 * alpha/beta (entry g of HOST arrays of scalars of the dtype; complex: (re,
 * im) pairs), DEVICE base pointers A[g], B[g], C[g] (held in HOST arrays),
 * ld's, strides and batch[g].  Each group is planned for its own size class
 * and enqueued in order on `stream`; every group is validated first, so on
 * any argument error nothing is enqueued.                                  */
iaat_status_t iaat_gemm_grouped_strided(
    iaat_dtype_t dtype, int64_t group_count, const char *transA, const char *transB,
    const int64_t *M, const int64_t *N, const int64_t *K, const void *alpha,
    const void *const *A, const int64_t *lda, const int64_t *strideA,
    const void *const *B, const int64_t *ldb, const int64_t *strideB,
    const void *beta, void *const *C, const int64_t *ldc, const int64_t *strideC,
    const int64_t *batch, void *stream);

/* Typed convenience wrappers (scalars by value). */
iaat_status_t iaat_sgemm_strided_batched(char transA, char transB, int64_t M, int64_t N,
    int64_t K, float alpha, const float *A, int64_t lda, int64_t strideA, const float *B,
    int64_t ldb, int64_t strideB, float beta, float *C, int64_t ldc, int64_t strideC,
    int64_t batch, void *stream);
iaat_status_t iaat_dgemm_strided_batched(char transA, char transB, int64_t M, int64_t N,
    int64_t K, double alpha, const double *A, int64_t lda, int64_t strideA, const double *B,
    int64_t ldb, int64_t strideB, double beta, double *C, int64_t ldc, int64_t strideC,
    int64_t batch, void *stream);
iaat_status_t iaat_sgemm_batched(char transA, char transB, int64_t M, int64_t N, int64_t K,
    float alpha, const float *const *Aarray, int64_t lda, const float *const *Barray,
    int64_t ldb, float beta, float *const *Carray, int64_t ldc, int64_t batch, void *stream);
iaat_status_t iaat_dgemm_batched(char transA, char transB, int64_t M, int64_t N, int64_t K,
    double alpha, const double *const *Aarray, int64_t lda, const double *const *Barray,
    int64_t ldb, double beta, double *const *Carray, int64_t ldc, int64_t batch, void *stream);

/* Complex typed wrappers: alpha / beta are host (re, im) pairs; A, B, C
 * interleaved complex (float2 / double2 per element). */
iaat_status_t iaat_cgemm_strided_batched(char transA, char transB, int64_t M, int64_t N,
    int64_t K, const float alpha[2], const float *A, int64_t lda, int64_t strideA, const float *B,
    int64_t ldb, int64_t strideB, const float beta[2], float *C, int64_t ldc, int64_t strideC,
    int64_t batch, void *stream);
iaat_status_t iaat_zgemm_strided_batched(char transA, char transB, int64_t M, int64_t N,
    int64_t K, const double alpha[2], const double *A, int64_t lda, int64_t strideA, const double *B,
    int64_t ldb, int64_t strideB, const double beta[2], double *C, int64_t ldc, int64_t strideC,
    int64_t batch, void *stream);

/* 1 if (transA, transB, M, N, K) is a small GEMM per PAPER.md:36, else 0.
 * Host only, no GPU needed.  Negative sizes -> 0.                          */
int iaat_is_small_gemm(char transA, char transB, int64_t M, int64_t N, int64_t K);

/* TN domain extension.  The paper bounds TN at cbrt(MNK) <= 32
 * because its NEON TN kernels cannot be vectorised; the
 * GPU kernels have no such limit.  iaat_set_tn_limit raises (or restores) the
 * M*N*K bound applied to transA='T', transB='N' calls, process-wide:
 * max_mnk in [32768, 512000], else IAAT_ERROR_INVALID_VALUE and the limit
 * is unchanged.  Default 32768 (the paper's domain).  iaat_is_small_gemm and
 * every GEMM entry point follow the current value.                        */
iaat_status_t iaat_set_tn_limit(int64_t max_mnk);
int64_t iaat_get_tn_limit(void);

/* Host only (no GPU needed): write, as JSON into json[0..cap), the plan the
 * strided call with these arguments would use (tile decomposition, tile
 * classes and their warps, problems per group, pipeline stages, grid, staging
 * mode, memops cost).  base_align_bytes = the common alignment of the A/B/C
 * base pointers (e.g. 4, 8, 16, 256); sm_count = the SM count to plan for
 * (148 on B200).  Returns IAAT_ERROR_INVALID_VALUE if cap is too small.   */
iaat_status_t iaat_plan_describe(
    iaat_dtype_t dtype, char transA, char transB, int64_t M, int64_t N, int64_t K,
    int64_t lda, int64_t strideA, int64_t ldb, int64_t strideB, int64_t ldc, int64_t strideC,
    int64_t batch, int beta_is_zero, int alpha_is_zero, int64_t base_align_bytes,
    int sm_count, char *json, size_t cap);

/* Host only (an ablation of the GPU planner): the paper's own
 * tiling of an SGEMM_NN M x N block with the Table I catalog
 * and the memops cost (m_0+n_0+...)K + 2MN as JSON:
 * mode 0 = Alg. 2 traced literally (readings DESIGN.md
 * A14), mode 1 = the exact optimum over Table I (Fig. 2's 72K+450 for
 * 15 x 15).  1 <= M, N <= 4096.                              */
iaat_status_t iaat_paper_tile(int mode, int64_t M, int64_t N, char *json, size_t cap);

/* Static description of the install-time kernel catalog as JSON. */
iaat_status_t iaat_catalog_describe(char *json, size_t cap);

const char *iaat_status_string(iaat_status_t status);

/* cudaError_t of the last IAAT_ERROR_CUDA on the calling thread (0 if none). */
int iaat_last_cuda_error(void);

/* Number of kernel launches the library has enqueued on this process (a
 * monotone counter, for benchmark bookkeeping). */
int64_t iaat_launch_count(void);

/* Library version, e.g. 100 for 0.1.0. */
int iaat_version(void);

#ifdef __cplusplus
}
#endif
#endif /* IAAT_H */
