// iaat_complex.cuh -- complex batched small GEMM (CGEMM / ZGEMM) on the slab
// family (the paper covers all four BLAS types: Table I C/Z rows,
// PAPER.md:96-97, the complex templates fcmla, and Eq. 2,
// 8 flops per complex multiply-add).
//
// Same staging as the real path (iaat_device.cuh: bulk copies of the
// verbatim interleaved (re, im) bytes of P problems, no pack pass), same
// exact tile classes and lane mapping; the micro-tile is complex:
//   acc(i,j) += opA(i,k) * opB(k,j)   k ascending, 4 real FMAs per complex MAC
//   fp32: (acc.re, acc.im) is one 64-bit register pair updated by two FFMA2
//         (fma.rn.f32x2): acc += (a.re, a.re) * (b.re, b.im)
//                         acc += (a.im, a.im) * (-b.im, b.re)
//   fp64: four DFMA: re += a.re*b.re; re -= a.im*b.im; im += a.re*b.im; im += a.im*b.re
// and the fused epilogue C = alpha*acc + beta*C_in with complex alpha, beta
// (C_in never read when beta == 0).
#pragma once
#include "iaat_device.cuh"

namespace iaat {

struct __align__(8) cf32 {
    float x, y;
};
struct __align__(16) cf64 {
    double x, y;
};
template <typename R> struct CplxOf;
template <> struct CplxOf<float> { typedef cf32 type; };
template <> struct CplxOf<double> { typedef cf64 type; };

// Complex register tile: fp32 as (re, im) 64-bit pairs (FFMA2), fp64 scalar.
template <typename R, int MR, int NR> struct CTile;

template <int MR, int NR>
struct CTile<float, MR, NR> {
    unsigned long long v[MR][NR];  // (re, im)
    __device__ __forceinline__ void zero()
    {
#pragma unroll
        for (int i = 0; i < MR; ++i)
#pragma unroll
            for (int j = 0; j < NR; ++j) v[i][j] = 0ull;
    }
    __device__ __forceinline__ void mac(const cf32 (&a)[MR], const cf32 (&b)[NR])
    {
#pragma unroll
        for (int j = 0; j < NR; ++j) {
            const unsigned long long b0 = pack_f32x2(b[j].x, b[j].y);
            const unsigned long long b1 = pack_f32x2(-b[j].y, b[j].x);
#pragma unroll
            for (int i = 0; i < MR; ++i) {
                ffma2(v[i][j], pack_f32x2(a[i].x, a[i].x), b0);
                ffma2(v[i][j], pack_f32x2(a[i].y, a[i].y), b1);
            }
        }
    }
    __device__ __forceinline__ void get(int i, int j, float &re, float &im) const { unpack_f32x2(v[i][j], re, im); }
};

template <int MR, int NR>
struct CTile<double, MR, NR> {
    double re[MR][NR], im[MR][NR];
    __device__ __forceinline__ void zero()
    {
#pragma unroll
        for (int i = 0; i < MR; ++i)
#pragma unroll
            for (int j = 0; j < NR; ++j) re[i][j] = im[i][j] = 0.0;
    }
    __device__ __forceinline__ void mac(const cf64 (&a)[MR], const cf64 (&b)[NR])
    {
#pragma unroll
        for (int j = 0; j < NR; ++j)
#pragma unroll
            for (int i = 0; i < MR; ++i) {
                re[i][j] = __fma_rn(a[i].x, b[j].x, re[i][j]);
                re[i][j] = __fma_rn(-a[i].y, b[j].y, re[i][j]);
                im[i][j] = __fma_rn(a[i].x, b[j].y, im[i][j]);
                im[i][j] = __fma_rn(a[i].y, b[j].x, im[i][j]);
            }
    }
    __device__ __forceinline__ void get(int i, int j, double &r, double &m) const
    {
        r = re[i][j];
        m = im[i][j];
    }
};

// acc(i,j) += sum_k opA(row0+i, k) * opB(k, col0+j), k ascending.
//   opA(i,k) = A[i + k*lda] (N) or A[k + i*lda] (T); opB(k,j) = B[k + j*ldb] (N) or B[j + k*ldb] (T)
// VEC (complex fp32 only, every address 16-byte aligned): two complex per
// 16-byte load -- two rows (tile-contiguous operand) or two k-steps
// (k-contiguous operand) -- in k-blocks of 2.
template <typename R, bool TA, bool TB, int MR, int NR, bool VEC>
__device__ __forceinline__ void cfma_tile(CTile<R, MR, NR> &acc, const typename CplxOf<R>::type *__restrict__ sA,
                                          const typename CplxOf<R>::type *__restrict__ sB, int lda, int ldb, int K,
                                          int row0, int col0)
{
    typedef typename CplxOf<R>::type CT;
    int k = 0;
    if (VEC && sizeof(CT) == 8) {
        // A tile-contiguous iff !TA; B tile-contiguous iff TB
        constexpr bool AV = !TA && (MR % 2 == 0), BV = TB && (NR % 2 == 0);
#pragma unroll 2
        for (; k + 2 <= K; k += 2) {
            CT a[2][MR], b[2][NR];
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
                if (AV) {
#pragma unroll
                    for (int i = 0; i < MR; i += 2) {
                        const float4 v = *reinterpret_cast<const float4 *>(sA + row0 + i + (k + kk) * lda);
                        a[kk][i] = CT{v.x, v.y};
                        a[kk][i + 1] = CT{v.z, v.w};
                    }
                } else if (!TA) {
#pragma unroll
                    for (int i = 0; i < MR; ++i) a[kk][i] = sA[row0 + i + (k + kk) * lda];
                }
                if (BV) {
#pragma unroll
                    for (int j = 0; j < NR; j += 2) {
                        const float4 v = *reinterpret_cast<const float4 *>(sB + col0 + j + (k + kk) * ldb);
                        b[kk][j] = CT{v.x, v.y};
                        b[kk][j + 1] = CT{v.z, v.w};
                    }
                } else if (TB) {
#pragma unroll
                    for (int j = 0; j < NR; ++j) b[kk][j] = sB[col0 + j + (k + kk) * ldb];
                }
            }
            if (TA) {  // k-contiguous: (k, k+1) of each row in one 16-byte load
#pragma unroll
                for (int i = 0; i < MR; ++i) {
                    const float4 v = *reinterpret_cast<const float4 *>(sA + k + (row0 + i) * lda);
                    a[0][i] = CT{v.x, v.y};
                    a[1][i] = CT{v.z, v.w};
                }
            }
            if (!TB) {
#pragma unroll
                for (int j = 0; j < NR; ++j) {
                    const float4 v = *reinterpret_cast<const float4 *>(sB + k + (col0 + j) * ldb);
                    b[0][j] = CT{v.x, v.y};
                    b[1][j] = CT{v.z, v.w};
                }
            }
            acc.mac(a[0], b[0]);
            acc.mac(a[1], b[1]);
        }
    }
#pragma unroll 4
    for (; k < K; ++k) {
        CT a[MR], b[NR];
#pragma unroll
        for (int i = 0; i < MR; ++i) a[i] = TA ? sA[k + (row0 + i) * lda] : sA[row0 + i + k * lda];
#pragma unroll
        for (int j = 0; j < NR; ++j) b[j] = TB ? sB[col0 + j + k * ldb] : sB[k + (col0 + j) * ldb];
        acc.mac(a, b);
    }
}

// C = alpha*acc + beta*C_in (complex), C_in loads of the tile issued before its stores.
template <typename R, int MR, int NR>
__device__ __forceinline__ void cepilogue(const CTile<R, MR, NR> &acc, typename CplxOf<R>::type *C,
                                          const typename CplxOf<R>::type *Cin, int ldc, int row0, int col0,
                                          R ar, R ai, R br, R bi, bool beta_zero, bool cin_global)
{
    typedef typename CplxOf<R>::type CT;
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        CT ci[MR];
        if (!beta_zero) {
#pragma unroll
            for (int i = 0; i < MR; ++i) {
                const CT *q = Cin + row0 + i + (int64_t)(col0 + j) * ldc;
                if (cin_global) {
                    ci[i].x = ldg_cs(&q->x);
                    ci[i].y = ldg_cs(&q->y);
                } else {
                    ci[i] = *q;
                }
            }
        }
#pragma unroll
        for (int i = 0; i < MR; ++i) {
            R sr, si;
            acc.get(i, j, sr, si);
            R tr = (R)0, tim = (R)0;
            if (!beta_zero) {
                tr = fma_rn(br, ci[i].x, mul_rn(-bi, ci[i].y));
                tim = fma_rn(br, ci[i].y, mul_rn(bi, ci[i].x));
            }
            CT o;
            o.x = fma_rn(ar, sr, fma_rn(-ai, si, tr));
            o.y = fma_rn(ar, si, fma_rn(ai, sr, tim));
            CT *c = C + row0 + i + (int64_t)(col0 + j) * ldc;
            stg_cs(&c->x, o.x);
            stg_cs(&c->y, o.y);
        }
    }
}

// One compute warp running complex tile class `c` over all groups of this CTA
// (the complex counterpart of fma_class_loop, same mapping and pipeline).
template <typename R, bool TA, bool TB, int MR, int NR, bool VEC = false>
__device__ __forceinline__ void cfma_class_loop(const IaatKParams &p, const IaatClass &c, unsigned char *smem,
                                                uint64_t *full, uint64_t *empty, int warp, int lane)
{
    typedef typename CplxOf<R>::type CT;
    int pl, ti, tj;
    bool tile_ok = true;
    if (c.bm == 0) {
        const int idx = (warp - c.warp_begin) * 32 + lane;
        pl = idx / c.tiles;
        const int t = idx - pl * c.tiles;
        ti = c.colfast ? t / c.tn : t % c.tm;
        tj = c.colfast ? t % c.tn : t / c.tm;
    } else {
        const int bn = 32 / c.bm;
        const int nbm = (c.tm + c.bm - 1) / c.bm, nbn = (c.tn + bn - 1) / bn;
        const int wb = warp - c.warp_begin;
        pl = wb / (nbm * nbn);
        const int blk = wb - pl * (nbm * nbn);
        ti = (blk % nbm) * c.bm + lane % c.bm;
        tj = (blk / nbm) * bn + lane / c.bm;
        tile_ok = ti < c.tm && tj < c.tn;
    }
    const int row0 = c.row_base + ti * MR, col0 = c.col_base + tj * NR;
    const R ar = (R)p.alpha, ai = (R)p.alpha_i, br = (R)p.beta, bi = (R)p.beta_i;
    const int64_t sab = p.sA * (int64_t)sizeof(CT), sbb = p.sB * (int64_t)sizeof(CT);
    const int64_t scb = p.sC * (int64_t)sizeof(CT);
    int it = 0;
    for (int64_t g = blockIdx.x; g < p.ngroups; g += gridDim.x, ++it) {
        const int s = it % p.S;
        const int64_t b0 = g * p.P;
        const int np = (int)min((int64_t)p.P, p.batch - b0);
        const bool active = tile_ok && pl < np;
        CTile<R, MR, NR> acc;
        acc.zero();
        mbar_wait(&full[s], (it / p.S) & 1);
        if (active) {
            StageView sv = stage_view(p, smem, s);
            const char *a_first = prob_ptr(p.A, p.Aarr, sab, b0);
            const char *b_first = prob_ptr(p.B, p.Barr, sbb, b0);
            const char *a_prob = p.modeA == IAAT_STAGE_SLAB ? a_first : prob_ptr(p.A, p.Aarr, sab, b0 + pl);
            const char *b_prob = p.modeB == IAAT_STAGE_SLAB ? b_first : prob_ptr(p.B, p.Barr, sbb, b0 + pl);
            const CT *sA = reinterpret_cast<const CT *>(sv.a + smem_offset(p.modeA, a_first, a_prob, sab, p.slotA, pl));
            const CT *sB = reinterpret_cast<const CT *>(sv.b + smem_offset(p.modeB, b_first, b_prob, sbb, p.slotB, pl));
            cfma_tile<R, TA, TB, MR, NR, VEC>(acc, sA, sB, p.lda, p.ldb, p.K, row0, col0);
        }
        if (!p.c_in_smem) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (active) {
            const char *c_first = prob_ptr(p.C, cptrs(p), scb, b0);
            const char *c_prob = prob_ptr(p.C, cptrs(p), scb, b0 + pl);
            CT *C = const_cast<CT *>(reinterpret_cast<const CT *>(c_prob));
            const CT *Cin = C;
            if (p.c_in_smem) {
                StageView sv = stage_view(p, smem, s);
                Cin = reinterpret_cast<const CT *>(sv.c + smem_offset(p.modeC, c_first, c_prob, scb, p.slotC, pl));
            }
            cepilogue<R, MR, NR>(acc, C, Cin, p.ldc, row0, col0, ar, ai, br, bi, p.beta_zero != 0, !p.c_in_smem);
        }
        if (p.c_in_smem) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
    }
}

// alpha == 0 or K == 0 path for complex C: C = beta*C (or zeros, C never read).
template <typename R>
__global__ void cscale_kernel(char *C, void *const *Carr, int64_t sC, int M, int N, int ldc, int64_t batch,
                              double br_d, double bi_d)
{
    typedef typename CplxOf<R>::type CT;
    const R br = (R)br_d, bi = (R)bi_d;
    const int64_t per = (int64_t)M * N;
    const int64_t total = per * batch;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = x / per;
        const int64_t e = x - b * per;
        const int j = (int)(e / M), i = (int)(e - (int64_t)j * M);
        CT *c = Carr ? reinterpret_cast<CT *>(Carr[b]) : reinterpret_cast<CT *>(C + b * sC * (int64_t)sizeof(CT));
        CT *q = c + i + (int64_t)j * ldc;
        CT o;
        if (br == (R)0 && bi == (R)0) {
            o.x = (R)0;
            o.y = (R)0;
        } else {
            const CT v = *q;
            o.x = fma_rn(br, v.x, mul_rn(-bi, v.y));
            o.y = fma_rn(br, v.y, mul_rn(bi, v.x));
        }
        *q = o;
    }
}

}  // namespace iaat
