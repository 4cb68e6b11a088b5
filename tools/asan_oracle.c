/* asan_oracle.c -- the C oracle (oracle/ref_gemm.c) under AddressSanitizer +
 * UndefinedBehaviorSanitizer: exact-fit buffers (no slack) for every
 * transposition, padded ld's, beta == 0 with C absent, alpha == 0, K == 0,
 * real and complex.  Built and run by tests/test_host_sanitizers.py. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

int iaat_ref_gemm(int dtype, char transA, char transB, int64_t M, int64_t N, int64_t K, double alpha,
                  const void *A, int64_t lda, int64_t strideA, const void *B, int64_t ldb, int64_t strideB,
                  double beta, const void *C, int64_t ldc, int64_t strideC, int64_t batch, double *ref, double *den,
                  int nthreads, int *used);
int iaat_ref_cgemm(int dtype, char transA, char transB, int64_t M, int64_t N, int64_t K, double alpha_re,
                   double alpha_im, const void *A, int64_t lda, int64_t strideA, const void *B, int64_t ldb,
                   int64_t strideB, double beta_re, double beta_im, const void *C, int64_t ldc, int64_t strideC,
                   int64_t batch, double *ref, double *den, int nthreads, int *used);

int main(void)
{
    const char tr[4][2] = {{'N', 'N'}, {'N', 'T'}, {'T', 'N'}, {'T', 'T'}};
    int calls = 0;
    for (int dt = 0; dt < 2; ++dt)
        for (int t = 0; t < 4; ++t)
            for (int M = 1; M <= 9; M += 4)
                for (int N = 1; N <= 9; N += 4)
                    for (int K = 0; K <= 9; K += 3)
                        for (int pad = 0; pad <= 2; pad += 2) {
                            const char tA = tr[t][0], tB = tr[t][1];
                            const int64_t ra = tA == 'N' ? M : K, ca = tA == 'N' ? K : M;
                            const int64_t rb = tB == 'N' ? K : N, cb = tB == 'N' ? N : K;
                            const int64_t lda = (ra > 0 ? ra : 1) + pad, ldb = (rb > 0 ? rb : 1) + pad,
                                          ldc = M + pad;
                            const int64_t batch = 3, sA = lda * ca, sB = ldb * cb, sC = ldc * N;
                            const size_t el = dt ? 8 : 4;
                            /* exact-fit allocations: the last problem ends at the buffer end */
                            const size_t nA = (size_t)((batch - 1) * sA + (ca ? (ca - 1) * lda + ra : 0));
                            const size_t nB = (size_t)((batch - 1) * sB + (cb ? (cb - 1) * ldb + rb : 0));
                            const size_t nC = (size_t)((batch - 1) * sC + (N - 1) * ldc + M);
                            char *A = malloc(nA * el + 1), *B = malloc(nB * el + 1), *C = malloc(nC * el);
                            for (size_t i = 0; i < nA * el; ++i) A[i] = 0;
                            for (size_t i = 0; i < nB * el; ++i) B[i] = 0;
                            for (size_t i = 0; i < nC * el; ++i) C[i] = 0;
                            double *ref = malloc(sizeof(double) * batch * M * N);
                            double *den = malloc(sizeof(double) * batch * M * N);
                            int used = 0;
                            for (int ab = 0; ab < 3; ++ab) {
                                const double alpha = ab == 2 ? 0.0 : 1.5, beta = ab == 1 ? 0.0 : 0.5;
                                if (iaat_ref_gemm(dt, tA, tB, M, N, K, alpha, A, lda, sA, B, ldb, sB, beta,
                                                  beta == 0.0 ? NULL : C, ldc, sC, batch, ref, den, 1, &used))
                                    return 1;
                                ++calls;
                            }
                            free(A);
                            free(B);
                            free(C);
                            free(ref);
                            free(den);
                        }
    printf("oracle calls %d\n", calls);
    return calls > 0 ? 0 : 1;
}
