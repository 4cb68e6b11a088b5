/*
 * oracle/ref_gemm.c -- CPU reference ("oracle") for batched small GEMM.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2208_09822_b200/) and includes nothing from it.
 *
 * What it computes (the plain definition; the method reaches exactly this
 * result up to rounding order, "C_c = A_c x B_c + C_c" on blocks
 * that partition C, "kernel executing plan"):
 *
 *   PAPER.md:30 (Sec. I)  "GEMM is used to compute C = alpha A x B + beta C.
 *                          Here C, A, B are M x N, M x K, and K x N matrices"
 *   PAPER.md:101 (Table I note) "NT means matrix A is not transposed and
 *                          matrix B is transposed ... We acquiescence the
 *                          matrix in column-major order."
 *
 * For every problem b and 0 <= i < M, 0 <= j < N:
 *   acc        = sum_{k=0..K-1} opA(i,k) * opB(k,j)      (k ascending, double)
 *   ref(i,j)   = alpha*acc + beta*Cin(i,j)               (double)
 *   den(i,j)   = |alpha| * sum_k |opA(i,k)|*|opB(k,j)| + |beta|*|Cin(i,j)|
 * with the BLAS quick-return readings of DESIGN.md (A3/A4): beta == 0 never
 * reads Cin (NaN in Cin does not propagate, its den term is 0); alpha == 0
 * never reads A or B.
 *
 * Storage (reading A1, BLAS convention): column-major,
 *   opA(i,k) = A[i + k*lda]   if transA == 'N'  (A stored M x K)
 *            = A[k + i*lda]   if transA == 'T'  (A stored K x M)
 *   opB(k,j) = B[k + j*ldb]   if transB == 'N'  (B stored K x N)
 *            = B[j + k*ldb]   if transB == 'T'  (B stored N x K)
 *   C(i,j)   = C[i + j*ldc]
 * Problem b's matrices start at X + b*strideX (elements).
 *
 * Outputs are packed double arrays: ref[b*M*N + i + j*M], den likewise.
 * fp32 inputs are widened to double; every fp32 x fp32 product is exact in
 * double (24+24 <= 53 significand bits), so the only rounding is the double
 * accumulation (|error| <= gamma_K * den).
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -shared -fPIC (no fast-math).
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

#ifdef _OPENMP
#include <omp.h>
#endif

static double load_elem(int dtype, const void *base, int64_t idx)
{
    if (dtype == 0)
        return (double)((const float *)base)[idx];
    return ((const double *)base)[idx];
}

/* opA(i,k) of problem b, PAPER.md:101 (transposition) + reading A1 (ld) */
static double opA(int dtype, char tA, const void *A, int64_t lda, int64_t off,
                  int64_t i, int64_t k)
{
    if (tA == 'N' || tA == 'n')
        return load_elem(dtype, A, off + i + k * lda);
    return load_elem(dtype, A, off + k + i * lda);
}

/* opB(k,j) of problem b */
static double opB(int dtype, char tB, const void *B, int64_t ldb, int64_t off,
                  int64_t k, int64_t j)
{
    if (tB == 'N' || tB == 'n')
        return load_elem(dtype, B, off + k + j * ldb);
    return load_elem(dtype, B, off + j + k * ldb);
}

/*
 * iaat_ref_gemm: returns 0 on success, -1 on bad arguments.
 *   dtype: 0 = fp32 inputs, 1 = fp64 inputs.
 *   Cin may be NULL when beta == 0.  den may be NULL.
 *   nthreads <= 0 means "OpenMP default"; the number actually used is
 *   written to *threads_used when that pointer is non-NULL.
 */
int iaat_ref_gemm(int dtype, char transA, char transB,
                  int64_t M, int64_t N, int64_t K, double alpha,
                  const void *A, int64_t lda, int64_t strideA,
                  const void *B, int64_t ldb, int64_t strideB,
                  double beta, const void *Cin, int64_t ldc, int64_t strideC,
                  int64_t batch, double *ref, double *den, int nthreads,
                  int *threads_used)
{
    if (dtype != 0 && dtype != 1) return -1;
    if (M < 0 || N < 0 || K < 0 || batch < 0) return -1;
    if (beta != 0.0 && Cin == NULL && M > 0 && N > 0) return -1;
    int used = 1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
    {
#pragma omp single
        used = omp_get_num_threads();
    }
#endif
    if (threads_used) *threads_used = used;

#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < batch; ++b) {
        const int64_t offA = b * strideA, offB = b * strideB, offC = b * strideC;
        double *r = ref + b * M * N;
        double *d = den ? den + b * M * N : NULL;
        for (int64_t j = 0; j < N; ++j) {
            for (int64_t i = 0; i < M; ++i) {
                double acc = 0.0, absacc = 0.0;
                if (alpha != 0.0) {                    /* reading A4 */
                    for (int64_t k = 0; k < K; ++k) {  /* k ascending */
                        double a = opA(dtype, transA, A, lda, offA, i, k);
                        double x = opB(dtype, transB, B, ldb, offB, k, j);
                        acc += a * x;
                        absacc += fabs(a) * fabs(x);
                    }
                }
                double out = alpha * acc;
                double dd = fabs(alpha) * absacc;
                if (beta != 0.0) {                     /* reading A3 */
                    double c = load_elem(dtype, Cin, offC + i + j * ldc);
                    out += beta * c;
                    dd += fabs(beta) * fabs(c);
                }
                r[i + j * M] = out;
                if (d) d[i + j * M] = dd;
            }
        }
    }
    return 0;
}

/*
 * iaat_ref_cgemm: the complex case (CGEMM / ZGEMM, Table I
 * rows, PAPER.md:156-171 complex templates, Eq. 2), same
 * definition over the complex field:
 *   acc      = sum_k opA(i,k) * opB(k,j)          (complex, k ascending, double)
 *   ref(i,j) = alpha*acc + beta*Cin(i,j)          (complex, double)
 *   den(i,j) = |alpha|_1 * sum_k |opA|_1*|opB|_1 + |beta|_1*|Cin|_1
 * where |x|_1 = |re x| + |im x| (a bound on every real product that enters
 * either component).  op is transposition only (N or T; no conjugation,
 * PAPER.md:101).  Elements are interleaved (re, im) pairs; ld's and strides
 * count complex elements.  dtype: 2 = complex fp32, 3 = complex fp64.
 * ref / den: packed, ref[2*(b*M*N + i + j*M) + {0,1}] = (re, im); den has
 * one real per element.
 */
static void load_c(int dtype, const void *base, int64_t idx, double *re, double *im)
{
    if (dtype == 2) {
        *re = (double)((const float *)base)[2 * idx];
        *im = (double)((const float *)base)[2 * idx + 1];
    } else {
        *re = ((const double *)base)[2 * idx];
        *im = ((const double *)base)[2 * idx + 1];
    }
}

int iaat_ref_cgemm(int dtype, char transA, char transB,
                   int64_t M, int64_t N, int64_t K, const double *alpha,
                   const void *A, int64_t lda, int64_t strideA,
                   const void *B, int64_t ldb, int64_t strideB,
                   const double *beta, const void *Cin, int64_t ldc, int64_t strideC,
                   int64_t batch, double *ref, double *den, int nthreads,
                   int *threads_used)
{
    if (dtype != 2 && dtype != 3) return -1;
    if (M < 0 || N < 0 || K < 0 || batch < 0) return -1;
    const double ar = alpha[0], ai = alpha[1], br = beta[0], bi = beta[1];
    const int beta_zero = (br == 0.0 && bi == 0.0), alpha_zero = (ar == 0.0 && ai == 0.0);
    if (!beta_zero && Cin == NULL && M > 0 && N > 0) return -1;
    const int tA = (transA == 'N' || transA == 'n') ? 0 : 1;
    const int tB = (transB == 'N' || transB == 'n') ? 0 : 1;
    int used = 1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
    {
#pragma omp single
        used = omp_get_num_threads();
    }
#endif
    if (threads_used) *threads_used = used;

#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < batch; ++b) {
        const int64_t offA = b * strideA, offB = b * strideB, offC = b * strideC;
        for (int64_t j = 0; j < N; ++j) {
            for (int64_t i = 0; i < M; ++i) {
                double sr = 0.0, si = 0.0, absacc = 0.0;
                if (!alpha_zero) {                         /* reading A4 */
                    for (int64_t k = 0; k < K; ++k) {      /* k ascending */
                        double xr, xi, yr, yi;
                        load_c(dtype, A, offA + (tA ? k + i * lda : i + k * lda), &xr, &xi);
                        load_c(dtype, B, offB + (tB ? j + k * ldb : k + j * ldb), &yr, &yi);
                        sr += xr * yr - xi * yi;           /* (x * y) re */
                        si += xr * yi + xi * yr;           /* (x * y) im */
                        absacc += (fabs(xr) + fabs(xi)) * (fabs(yr) + fabs(yi));
                    }
                }
                double outr = ar * sr - ai * si, outi = ar * si + ai * sr;
                double dd = (fabs(ar) + fabs(ai)) * absacc;
                if (!beta_zero) {                          /* reading A3 */
                    double cr, ci;
                    load_c(dtype, Cin, offC + i + j * ldc, &cr, &ci);
                    outr += br * cr - bi * ci;
                    outi += br * ci + bi * cr;
                    dd += (fabs(br) + fabs(bi)) * (fabs(cr) + fabs(ci));
                }
                const int64_t o = b * M * N + i + j * M;
                ref[2 * o] = outr;
                ref[2 * o + 1] = outi;
                if (den) den[o] = dd;
            }
        }
    }
    return 0;
}

/*
 * Small-GEMM predicate, PAPER.md:36 (Sec. I): "cbrt(MNK) <= 80 when
 * transposition ... is not TN, or cbrt(MNK) <= 32 when ... TN", evaluated as
 * the integer test M*N*K <= 80^3 (32^3) (reading A10, inclusive).
 */
int iaat_ref_is_small(char transA, char transB, int64_t M, int64_t N, int64_t K)
{
    int tn = (transA == 'T' || transA == 't') && (transB == 'N' || transB == 'n');
    int64_t lim = tn ? (int64_t)32 * 32 * 32 : (int64_t)80 * 80 * 80;
    if (M < 0 || N < 0 || K < 0) return 0;
    if (M == 0 || N == 0 || K == 0) return 1;
    if (M > lim || N > lim || K > lim) return 0;
    /* each factor <= 512000, so the product (< 1.4e17) cannot overflow */
    return M * N * K <= lim;
}
