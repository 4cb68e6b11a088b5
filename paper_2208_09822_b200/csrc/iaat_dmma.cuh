// iaat_dmma.cuh -- fp64 warp tiles on the DMMA tensor-core path.
//
// fp64 is a genuine dense contraction, and on sm_100a the only FP64
// tensor-core instruction is the legacy warp-level mma.sync.m8n8k4.f64
// (SASS DMMA.8x8x4; tcgen05 has no f64 kind).  A warp owns a
// (8*WM) x (8*WN) block of C and accumulates it in registers over the whole K
// of the problem -- the warp-level analogue of the paper's register-blocked
// kernel (Alg. 1: Cregs hold the whole C_c block while
// columns of A_c and rows of B_c stream through).
//
// The MMA is issued in transposed form, D' = op(B)^T op(A)^T (= C^T), so a
// lane's two accumulator elements are two CONSECUTIVE ROWS of one column of
// the column-major C (one 16-byte store) -- PAPER.md:312 "SIMD friendly".
//   A' fragment (8x4, row): lane (g = lane/4, t = lane%4) holds
//        A'(g, t) = op(B)(k0+t, col0+g)
//   B' fragment (4x8, col): lane holds B'(t, g) = op(A)(row0+g, k0+t)
//   D' (8x8): lane holds D'(g, 2t+h) = C(row0 + 2t + h, col0 + g), h = 0, 1
// K % 8 tail: the missing k of the last steps are zero in BOTH fragments
// (0*0 adds nothing); no MMA is predicated.
#pragma once
#include "iaat_device.cuh"

namespace iaat {

__device__ __forceinline__ void dmma_8x8x4(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// K is consumed 8 at a time as two DMMA k-steps.  The MMA sums its 4
// k-positions in any order, so position t of step h is given the actual k
// k0 + 2t + h (the same for every row/column -- consistent between the two
// fragments): a lane's two k-values are ADJACENT, and for an operand that is
// contiguous along k one 16-byte load (LDS.128) feeds both steps.
template <bool KCONTIG, bool VEC>
__device__ __forceinline__ void dmma_pair(const double *__restrict__ X, int off, int ld, int k0, int t, int K,
                                          bool full, double &v0, double &v1)
{
    const int k = k0 + 2 * t;
    if (KCONTIG) {
        const double *p = X + off + k;  // element (k, r) at X[k + r*ld], off = r*ld
        if (full) {
            if (VEC) {
                double2 d = *reinterpret_cast<const double2 *>(p);
                v0 = d.x;
                v1 = d.y;
            } else {
                v0 = p[0];
                v1 = p[1];
            }
        } else {
            v0 = k < K ? p[0] : 0.0;
            v1 = k + 1 < K ? p[1] : 0.0;
        }
    } else {
        const double *p = X + off + (int64_t)k * ld;  // element (r, k) at X[r + k*ld], off = r
        if (full) {
            v0 = p[0];
            v1 = p[ld];
        } else {
            v0 = k < K ? p[0] : 0.0;
            v1 = k + 1 < K ? p[ld] : 0.0;
        }
    }
}

template <bool TA, bool TB, int WM, int WN, bool VEC>
__device__ __forceinline__ void dmma_tile(double (&acc)[WM][WN][2], const double *__restrict__ sA,
                                          const double *__restrict__ sB, int lda, int ldb, int K,
                                          int row0, int col0, int g, int t)
{
    // op(A)(i,k): TA ? A[k + i*lda] (k-contiguous) : A[i + k*lda]
    // op(B)(k,j): TB ? B[j + k*ldb] : B[k + j*ldb] (k-contiguous)
    int aoff[WM], boff[WN];
#pragma unroll
    for (int mi = 0; mi < WM; ++mi) {
        const int r = row0 + 8 * mi + g;
        aoff[mi] = TA ? r * lda : r;
    }
#pragma unroll
    for (int nj = 0; nj < WN; ++nj) {
        const int cidx = col0 + 8 * nj + g;
        boff[nj] = TB ? cidx : cidx * ldb;
    }
    const int kfull = K & ~7;
#pragma unroll 1
    for (int k0 = 0; k0 < K; k0 += 8) {
        const bool full = k0 < kfull;
        double af[WM][2], bf[WN][2];
#pragma unroll
        for (int mi = 0; mi < WM; ++mi) dmma_pair<TA, VEC>(sA, aoff[mi], lda, k0, t, K, full, af[mi][0], af[mi][1]);
#pragma unroll
        for (int nj = 0; nj < WN; ++nj) dmma_pair<!TB, VEC>(sB, boff[nj], ldb, k0, t, K, full, bf[nj][0], bf[nj][1]);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int mi = 0; mi < WM; ++mi)
#pragma unroll
                for (int nj = 0; nj < WN; ++nj)
                    dmma_8x8x4(acc[mi][nj][0], acc[mi][nj][1], bf[nj][h], af[mi][h]);
    }
}

// One compute warp running DMMA class `c`: the class' warps share the
// group's (problem, warp-tile) items round-robin.
template <bool TA, bool TB, int WM, int WN, bool VEC>
__device__ __forceinline__ void dmma_class_loop(const IaatKParams &p, const IaatClass &c,
                                                unsigned char *smem, uint64_t *full,
                                                uint64_t *empty, int warp, int lane)
{
    const int g = lane >> 2, t = lane & 3;
    const int nw = c.warp_end - c.warp_begin, wi = warp - c.warp_begin;
    const double alpha = p.alpha, beta = p.beta;
    const int64_t sab = p.sA * 8, sbb = p.sB * 8, scb = p.sC * 8;
    int it = 0;
    for (int64_t gr = blockIdx.x; gr < p.ngroups; gr += gridDim.x, ++it) {
        const int s = it % p.S;
        const int64_t b0 = gr * p.P;
        const int np = (int)min((int64_t)p.P, p.batch - b0);
        mbar_wait(&full[s], (it / p.S) & 1);
        StageView sv = stage_view(p, smem, s);
        const char *a_first = prob_ptr(p.A, p.Aarr, sab, b0);
        const char *b_first = prob_ptr(p.B, p.Barr, sbb, b0);
        const int items = np * c.tiles;
        for (int item = wi; item < items; item += nw) {
            const int pl = item / c.tiles, tt = item - pl * c.tiles;
            const int ti = c.colfast ? tt / c.tn : tt % c.tm;
            const int tj = c.colfast ? tt % c.tn : tt / c.tm;
            const int row0 = c.row_base + ti * 8 * WM, col0 = c.col_base + tj * 8 * WN;
            const char *a_prob = p.modeA == IAAT_STAGE_SLAB ? a_first : prob_ptr(p.A, p.Aarr, sab, b0 + pl);
            const char *b_prob = p.modeB == IAAT_STAGE_SLAB ? b_first : prob_ptr(p.B, p.Barr, sbb, b0 + pl);
            const double *sA = reinterpret_cast<const double *>(
                sv.a + smem_offset(p.modeA, a_first, a_prob, sab, p.slotA, pl));
            const double *sB = reinterpret_cast<const double *>(
                sv.b + smem_offset(p.modeB, b_first, b_prob, sbb, p.slotB, pl));
            double acc[WM][WN][2];
#pragma unroll
            for (int mi = 0; mi < WM; ++mi)
#pragma unroll
                for (int nj = 0; nj < WN; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
            dmma_tile<TA, TB, WM, WN, VEC>(acc, sA, sB, p.lda, p.ldb, p.K, row0, col0, g, t);
            const char *c_first = prob_ptr(p.C, cptrs(p), scb, b0);
            const char *c_prob = prob_ptr(p.C, cptrs(p), scb, b0 + pl);
            double *C = const_cast<double *>(reinterpret_cast<const double *>(c_prob));
            const double *Cin = C;
            if (p.c_in_smem)
                Cin = reinterpret_cast<const double *>(
                    sv.c + smem_offset(p.modeC, c_first, c_prob, scb, p.slotC, pl));
#pragma unroll
            for (int mi = 0; mi < WM; ++mi)
#pragma unroll
                for (int nj = 0; nj < WN; ++nj) {
                    const int64_t eo = (row0 + 8 * mi + 2 * t) + (int64_t)(col0 + 8 * nj + g) * p.ldc;
                    double *cp = C + eo;
                    const double *cip = Cin + eo;
                    double o[2];
                    if (VEC) {
                        if (p.beta_zero) {
                            o[0] = mul_rn(alpha, acc[mi][nj][0]);
                            o[1] = mul_rn(alpha, acc[mi][nj][1]);
                        } else {
                            double ci[2];
                            ld_vec<double>(cip, ci);
                            o[0] = fma_rn(alpha, acc[mi][nj][0], mul_rn(beta, ci[0]));
                            o[1] = fma_rn(alpha, acc[mi][nj][1], mul_rn(beta, ci[1]));
                        }
                        st_vec<double>(cp, o);
                    } else {
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            cp[h] = p.beta_zero ? mul_rn(alpha, acc[mi][nj][h])
                                                : fma_rn(alpha, acc[mi][nj][h], mul_rn(beta, cip[h]));
                    }
                }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
}

}  // namespace iaat
