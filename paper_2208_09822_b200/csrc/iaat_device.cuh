// iaat_device.cuh -- sm_100a device code of the batched small-GEMM path.
//
// One persistent launch per call ("kernel executing plan").
// Each CTA loops over groups of P consecutive problems:
//   producer warp : HBM -> SMEM staging of the group's A and B with
//                   cp.async.bulk (UBLKCP) into an S-stage mbarrier ring, the
//                   bytes copied verbatim in their global layout -- NO pack
//                   pass (the pack step is what IAAT
//                   removes).
//   compute warps : every warp runs ONE exact-size micro-tile class (the GPU
//                   analogue of the paper's fixed-size kernels, PAPER.md:105,
//                   179 "C_c = A_c x B_c + C_c"), so no lane executes
//                   predicated boundary code.  Lanes map
//                   to (problem, tile).  The k loop is a chain of rank-1
//                   updates, one FMA per (i, j, k), k ascending (PAPER.md:
//                   185-213, Alg. 1), and the alpha/beta epilogue is fused.
//
// fp32 runs on FFMA (IEEE fp32, no TF32); fp64 on DFMA here and on DMMA in
// iaat_dmma.cuh.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "iaat_params.h"

namespace iaat {

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    while (!mbar_try_wait(bar, parity)) {
    }
}

// 1-D bulk async copy global -> shared (SASS UBLKCP.S.G); completion is
// signalled as transaction bytes on `bar`.  dst, src, bytes: multiples of 16.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar, uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ unsigned warp_sum(unsigned v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ------------------------------------------------------------------ vectors
template <typename T> struct VecOf;
template <> struct VecOf<float> {
    static constexpr int W = 4;
    typedef float4 type;
};
template <> struct VecOf<double> {
    static constexpr int W = 2;
    typedef double2 type;
};

template <typename T>
__device__ __forceinline__ void ld_vec(const T *p, T *out)
{
    typedef typename VecOf<T>::type V;
    V v = *reinterpret_cast<const V *>(p);
    const T *e = reinterpret_cast<const T *>(&v);
#pragma unroll
    for (int w = 0; w < VecOf<T>::W; ++w) out[w] = e[w];
}

template <typename T>
__device__ __forceinline__ void st_vec(T *p, const T *in)
{
    typedef typename VecOf<T>::type V;
    V v;
    T *e = reinterpret_cast<T *>(&v);
#pragma unroll
    for (int w = 0; w < VecOf<T>::W; ++w) e[w] = in[w];
    *reinterpret_cast<V *>(p) = v;
}

// Global-space streaming accesses for C (ld/st.global.cs): C is touched
// once per call, so it should not displace operands in L2; the explicit
// space also avoids generic LD/ST.
__device__ __forceinline__ float ldg_cs(const float *p) { return __ldcs(p); }
__device__ __forceinline__ double ldg_cs(const double *p) { return __ldcs(p); }
__device__ __forceinline__ void stg_cs(float *p, float v) { __stcs(p, v); }
__device__ __forceinline__ void stg_cs(double *p, double v) { __stcs(p, v); }

template <typename T>
__device__ __forceinline__ void ldg_vec_cs(const T *p, T *out)
{
    typedef typename VecOf<T>::type V;
    V v = __ldcs(reinterpret_cast<const V *>(p));
    const T *e = reinterpret_cast<const T *>(&v);
#pragma unroll
    for (int w = 0; w < VecOf<T>::W; ++w) out[w] = e[w];
}

template <typename T>
__device__ __forceinline__ void stg_vec_cs(T *p, const T *in)
{
    typedef typename VecOf<T>::type V;
    V v;
    T *e = reinterpret_cast<T *>(&v);
#pragma unroll
    for (int w = 0; w < VecOf<T>::W; ++w) e[w] = in[w];
    __stcs(reinterpret_cast<V *>(p), v);
}

__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

// ------------------------------------------------------------------ register tile
// The C_c register block of one lane (Cregs) with the
// rank-1 update acc(i,j) += a(i) * b(j).  fp32 tiles are held as 64-bit
// register pairs and updated with FFMA2 (fma.rn.f32x2, sm_100a: two
// independent IEEE fp32 FMAs per instruction -- bitwise the same as two
// FFMAs, half the issue slots); the scalar operand is a broadcast that ptxas
// folds into the instruction (Rn.F32).  PAIR: 1 = pairs along i (the a
// fragment arrives as consecutive registers from a 16-byte load), 2 = pairs
// along j, 0 = scalar FMAs (fp64, or no even dimension).
__device__ __forceinline__ unsigned long long pack_f32x2(float lo, float hi)
{
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}

__device__ __forceinline__ void unpack_f32x2(unsigned long long v, float &lo, float &hi)
{
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}

__device__ __forceinline__ void ffma2(unsigned long long &c, unsigned long long a, unsigned long long b)
{
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(a), "l"(b));
}

template <typename T, int MR, int NR, int PAIR>
struct RegTile {
    T v[MR][NR];
    __device__ __forceinline__ void zero()
    {
#pragma unroll
        for (int i = 0; i < MR; ++i)
#pragma unroll
            for (int j = 0; j < NR; ++j) v[i][j] = (T)0;
    }
    template <typename AF, typename BF>
    __device__ __forceinline__ void rank1(const AF &a, const BF &b)
    {
#pragma unroll
        for (int j = 0; j < NR; ++j)
#pragma unroll
            for (int i = 0; i < MR; ++i) v[i][j] = fma_rn(a(i), b(j), v[i][j]);
    }
    __device__ __forceinline__ void get(T (&o)[MR][NR]) const
    {
#pragma unroll
        for (int i = 0; i < MR; ++i)
#pragma unroll
            for (int j = 0; j < NR; ++j) o[i][j] = v[i][j];
    }
};

template <int MR, int NR>
struct RegTile<float, MR, NR, 1> {  // pairs (i, i+1)
    unsigned long long v[MR / 2][NR];
    __device__ __forceinline__ void zero()
    {
#pragma unroll
        for (int i = 0; i < MR / 2; ++i)
#pragma unroll
            for (int j = 0; j < NR; ++j) v[i][j] = 0ull;
    }
    template <typename AF, typename BF>
    __device__ __forceinline__ void rank1(const AF &a, const BF &b)
    {
#pragma unroll
        for (int j = 0; j < NR; ++j) {
            const unsigned long long bb = pack_f32x2(b(j), b(j));
#pragma unroll
            for (int i = 0; i < MR / 2; ++i) ffma2(v[i][j], pack_f32x2(a(2 * i), a(2 * i + 1)), bb);
        }
    }
    __device__ __forceinline__ void get(float (&o)[MR][NR]) const
    {
#pragma unroll
        for (int i = 0; i < MR / 2; ++i)
#pragma unroll
            for (int j = 0; j < NR; ++j) unpack_f32x2(v[i][j], o[2 * i][j], o[2 * i + 1][j]);
    }
};

template <int MR, int NR>
struct RegTile<float, MR, NR, 2> {  // pairs (j, j+1)
    unsigned long long v[MR][NR / 2];
    __device__ __forceinline__ void zero()
    {
#pragma unroll
        for (int i = 0; i < MR; ++i)
#pragma unroll
            for (int j = 0; j < NR / 2; ++j) v[i][j] = 0ull;
    }
    template <typename AF, typename BF>
    __device__ __forceinline__ void rank1(const AF &a, const BF &b)
    {
#pragma unroll
        for (int j = 0; j < NR / 2; ++j) {
            const unsigned long long bb = pack_f32x2(b(2 * j), b(2 * j + 1));
#pragma unroll
            for (int i = 0; i < MR; ++i) ffma2(v[i][j], pack_f32x2(a(i), a(i)), bb);
        }
    }
    __device__ __forceinline__ void get(float (&o)[MR][NR]) const
    {
#pragma unroll
        for (int i = 0; i < MR; ++i)
#pragma unroll
            for (int j = 0; j < NR / 2; ++j) unpack_f32x2(v[i][j], o[i][2 * j], o[i][2 * j + 1]);
    }
};

template <int MR, int NR>
struct RegTile<float, MR, NR, 3> {  // odd MR: pairs (i, i+1) for i < MR - 1, the last row scalar
    unsigned long long v[MR / 2][NR];
    float t[NR];
    __device__ __forceinline__ void zero()
    {
#pragma unroll
        for (int j = 0; j < NR; ++j) {
#pragma unroll
            for (int i = 0; i < MR / 2; ++i) v[i][j] = 0ull;
            t[j] = 0.f;
        }
    }
    template <typename AF, typename BF>
    __device__ __forceinline__ void rank1(const AF &a, const BF &b)
    {
#pragma unroll
        for (int j = 0; j < NR; ++j) {
            const float bj = b(j);
            const unsigned long long bb = pack_f32x2(bj, bj);
#pragma unroll
            for (int i = 0; i < MR / 2; ++i) ffma2(v[i][j], pack_f32x2(a(2 * i), a(2 * i + 1)), bb);
            t[j] = fma_rn(a(MR - 1), bj, t[j]);
        }
    }
    __device__ __forceinline__ void get(float (&o)[MR][NR]) const
    {
#pragma unroll
        for (int j = 0; j < NR; ++j) {
#pragma unroll
            for (int i = 0; i < MR / 2; ++i) unpack_f32x2(v[i][j], o[2 * i][j], o[2 * i + 1][j]);
            o[MR - 1][j] = t[j];
        }
    }
};

template <int MR, int NR>
struct RegTile<float, MR, NR, 4> {  // odd NR: pairs (j, j+1) for j < NR - 1, the last column scalar
    unsigned long long v[MR][NR / 2];
    float t[MR];
    __device__ __forceinline__ void zero()
    {
#pragma unroll
        for (int i = 0; i < MR; ++i) {
#pragma unroll
            for (int j = 0; j < NR / 2; ++j) v[i][j] = 0ull;
            t[i] = 0.f;
        }
    }
    template <typename AF, typename BF>
    __device__ __forceinline__ void rank1(const AF &a, const BF &b)
    {
#pragma unroll
        for (int j = 0; j < NR / 2; ++j) {
            const unsigned long long bb = pack_f32x2(b(2 * j), b(2 * j + 1));
#pragma unroll
            for (int i = 0; i < MR; ++i) ffma2(v[i][j], pack_f32x2(a(i), a(i)), bb);
        }
#pragma unroll
        for (int i = 0; i < MR; ++i) t[i] = fma_rn(a(i), b(NR - 1), t[i]);
    }
    __device__ __forceinline__ void get(float (&o)[MR][NR]) const
    {
#pragma unroll
        for (int i = 0; i < MR; ++i) {
#pragma unroll
            for (int j = 0; j < NR / 2; ++j) unpack_f32x2(v[i][j], o[i][2 * j], o[i][2 * j + 1]);
            o[i][NR - 1] = t[i];
        }
    }
};

// Element (i, j) of a register tile, i and j compile-time after unrolling
// (a pair's unpack is a register rename).
template <int MR, int NR, int PAIR>
__device__ __forceinline__ float tile_at(const RegTile<float, MR, NR, PAIR> &t, int i, int j)
{
    float lo, hi;
    if constexpr (PAIR == 0) {
        return t.v[i][j];
    } else if constexpr (PAIR == 1 || PAIR == 3) {
        if constexpr (PAIR == 3) {
            if (i == MR - 1) return t.t[j];
        }
        unpack_f32x2(t.v[i / 2][j], lo, hi);
        return (i & 1) ? hi : lo;
    } else {
        if constexpr (PAIR == 4) {
            if (j == NR - 1) return t.t[i];
        }
        unpack_f32x2(t.v[i][j / 2], lo, hi);
        return (j & 1) ? hi : lo;
    }
}

// Pairing choice: along the dimension whose fragment arrives as consecutive
// registers (contiguous in smem); fp64 and odd tiles use scalar FMAs.
template <typename T, bool A_CONTIG, bool B_CONTIG, int MR, int NR>
struct PairOf {
    static constexpr int value = sizeof(T) != 4 ? 0 : (A_CONTIG && MR % 2 == 0) ? 1 : (B_CONTIG && NR % 2 == 0) ? 2 : 0;
};

// ------------------------------------------------------------------ smem layout
struct StageView {
    unsigned char *a;  // this stage's A region
    unsigned char *b;  // this stage's B region
    unsigned char *c;  // this stage's C_in region (c_in_smem only)
};

__device__ __forceinline__ StageView stage_view(const IaatKParams &p, unsigned char *smem, int s)
{
    unsigned char *base = smem + IAAT_BAR_BYTES + (size_t)s * p.stage_bytes;
    return StageView{base, base + p.capA, base + p.capA + p.capB};
}

// Global byte address of problem b's operand (strided or pointer-array API).
__device__ __forceinline__ const char *prob_ptr(const char *base, const void *const *arr,
                                                int64_t stride_bytes, int64_t b)
{
    return arr ? reinterpret_cast<const char *>(arr[b]) : base + b * stride_bytes;
}

__device__ __forceinline__ const void *const *cptrs(const IaatKParams &p)
{
    return reinterpret_cast<const void *const *>(p.Carr);
}

// Byte offset, inside the stage region, of local problem pl's operand.
__device__ __forceinline__ int smem_offset(int mode, const char *group_first, const char *prob,
                                           int64_t stride_bytes, int slot, int pl)
{
    if (mode == IAAT_STAGE_SLAB)
        return (int)(reinterpret_cast<uintptr_t>(group_first) & 15) + (int)(pl * stride_bytes);
    return pl * slot + (int)(reinterpret_cast<uintptr_t>(prob) & 15);
}

// ------------------------------------------------------------------ producer
// One warp.  SLAB mode: lane 0 copies the 16 B-aligned enclosing span of the
// group's operand (over-read <= 15 B per end, inside the same 16 B granule as
// valid data, so it can never touch an unmapped page); PERPROB mode: lanes
// copy one problem each.  Bytes are moved verbatim (no pack, no convert).
template <typename T>
__device__ __forceinline__ unsigned stage_operand(bool issue, int mode, const char *base,
                                                  const void *const *arr, int64_t stride_el,
                                                  int span, int slot, int64_t b0, int np,
                                                  unsigned char *dst, uint64_t *bar,
                                                  uint64_t pol, int lane)
{
    const int64_t sb = stride_el * (int64_t)sizeof(T);
    unsigned bytes = 0;
    if (mode == IAAT_STAGE_SLAB) {
        if (lane == 0) {
            const char *first = prob_ptr(base, arr, sb, b0);
            uintptr_t lo = reinterpret_cast<uintptr_t>(first) & ~(uintptr_t)15;
            uintptr_t hi = (reinterpret_cast<uintptr_t>(first) + (uintptr_t)((np - 1) * sb) +
                            (uintptr_t)span + 15) & ~(uintptr_t)15;
            bytes = (unsigned)(hi - lo);
            if (issue) bulk_g2s(dst, reinterpret_cast<const void *>(lo), bytes, bar, pol);
        }
    } else {
        for (int pl = lane; pl < np; pl += 32) {
            const char *pp = prob_ptr(base, arr, sb, b0 + pl);
            uintptr_t lo = reinterpret_cast<uintptr_t>(pp) & ~(uintptr_t)15;
            uintptr_t hi = (reinterpret_cast<uintptr_t>(pp) + (uintptr_t)span + 15) & ~(uintptr_t)15;
            unsigned nb = (unsigned)(hi - lo);
            bytes += nb;
            if (issue) bulk_g2s(dst + pl * slot, reinterpret_cast<const void *>(lo), nb, bar, pol);
        }
    }
    return bytes;
}

template <typename T>
__device__ void producer_loop(const IaatKParams &p, unsigned char *smem, uint64_t *full,
                              uint64_t *empty, int lane)
{
    const uint64_t pol = policy_evict_first();
    int it = 0;
    for (int64_t g = blockIdx.x; g < p.ngroups; g += gridDim.x, ++it) {
        const int s = it % p.S;
        if (it >= p.S) mbar_wait(&empty[s], ((it / p.S) - 1) & 1);
        const int64_t b0 = g * p.P;
        const int np = (int)min((int64_t)p.P, p.batch - b0);
        StageView sv = stage_view(p, smem, s);
        // pass 1: count bytes, arm the barrier; pass 2: issue the copies
        const void *const *carr = reinterpret_cast<const void *const *>(p.Carr);
        unsigned bytes = stage_operand<T>(false, p.modeA, p.A, p.Aarr, p.sA, p.spanA, p.slotA,
                                          b0, np, sv.a, &full[s], pol, lane) +
                         stage_operand<T>(false, p.modeB, p.B, p.Barr, p.sB, p.spanB, p.slotB,
                                          b0, np, sv.b, &full[s], pol, lane);
        if (p.c_in_smem)
            bytes += stage_operand<T>(false, p.modeC, p.C, carr, p.sC, p.spanC, p.slotC, b0, np,
                                      sv.c, &full[s], pol, lane);
        bytes = warp_sum(bytes);
        if (lane == 0) mbar_arrive_expect_tx(&full[s], bytes);
        __syncwarp();
        stage_operand<T>(true, p.modeA, p.A, p.Aarr, p.sA, p.spanA, p.slotA, b0, np, sv.a,
                         &full[s], pol, lane);
        stage_operand<T>(true, p.modeB, p.B, p.Barr, p.sB, p.spanB, p.slotB, b0, np, sv.b,
                         &full[s], pol, lane);
        if (p.c_in_smem)
            stage_operand<T>(true, p.modeC, p.C, carr, p.sC, p.spanC, p.slotC, b0, np, sv.c,
                             &full[s], pol, lane);
        if (p.prefetch_c) {
            // C_in will be read by the epilogue: warm L2 now (no smem needed)
            const int64_t scb = p.sC * (int64_t)sizeof(T);
            const int cspan = (int)(((int64_t)(p.N - 1) * p.ldc + p.M) * (int64_t)sizeof(T));
            if (p.Carr == nullptr) {
                if (lane == 0) {
                    const char *first = p.C + b0 * scb;
                    uintptr_t lo = reinterpret_cast<uintptr_t>(first) & ~(uintptr_t)15;
                    uintptr_t hi = (reinterpret_cast<uintptr_t>(first) + (uintptr_t)((np - 1) * scb) +
                                    (uintptr_t)cspan + 15) & ~(uintptr_t)15;
                    bulk_prefetch_l2(reinterpret_cast<const void *>(lo), (uint32_t)(hi - lo));
                }
            } else {
                for (int pl = lane; pl < np; pl += 32) {
                    const char *pp = reinterpret_cast<const char *>(p.Carr[b0 + pl]);
                    uintptr_t lo = reinterpret_cast<uintptr_t>(pp) & ~(uintptr_t)15;
                    uintptr_t hi = (reinterpret_cast<uintptr_t>(pp) + (uintptr_t)cspan + 15) & ~(uintptr_t)15;
                    bulk_prefetch_l2(reinterpret_cast<const void *>(lo), (uint32_t)(hi - lo));
                }
            }
        }
    }
}

// ------------------------------------------------------------------ FMA micro-tile
// Loads of one k-block (KU = 4 k-steps) of op(A) rows row0..row0+MR-1 and of
// op(B) columns col0..col0+NR-1 from the staged (unpacked) problem.
//   op(A)(i,k) = A[i + k*lda] (N: contiguous along the tile)
//              = A[k + i*lda] (T: contiguous along k)
//   op(B)(k,j) = B[k + j*ldb] (N: contiguous along k)
//              = B[j + k*ldb] (T: contiguous along the tile)
// VEC: 16-byte vector loads along the contiguous direction (the paper's
// "SIMD friendly" principle); the planner only sets it when
// every address involved is 16 B aligned.
// KU = k-steps per unrolled block = one 16-byte vector along k.
template <typename T> struct KUnroll { static constexpr int value = VecOf<T>::W; };

template <typename T, bool TRANS_TILE_CONTIG, int R, bool VEC>
__device__ __forceinline__ void load_frag(T (&f)[KUnroll<T>::value][R], const T *X, int ld, int k,
                                          int r0)
{
    constexpr int W = VecOf<T>::W;
    constexpr int KU = KUnroll<T>::value;
    if (!TRANS_TILE_CONTIG) {
        // contiguous along the tile dim: element (r, k) at X[r + k*ld]
        if (VEC && (R % W) == 0) {
#pragma unroll
            for (int kk = 0; kk < KU; ++kk)
#pragma unroll
                for (int q = 0; q < R / W; ++q) ld_vec<T>(X + r0 + q * W + (k + kk) * ld, &f[kk][q * W]);
        } else {
#pragma unroll
            for (int kk = 0; kk < KU; ++kk)
#pragma unroll
                for (int r = 0; r < R; ++r) f[kk][r] = X[r0 + r + (k + kk) * ld];
        }
    } else {
        // contiguous along k: element (r, k) at X[k + r*ld]
        if (VEC) {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int q = 0; q < KU / W; ++q) {
                    T t[W];
                    ld_vec<T>(X + k + q * W + (r0 + r) * ld, t);
#pragma unroll
                    for (int w = 0; w < W; ++w) f[q * W + w][r] = t[w];
                }
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int kk = 0; kk < KU; ++kk) f[kk][r] = X[k + kk + (r0 + r) * ld];
        }
    }
}

// Single k-step (scalar) load for the K % KU remainder.
template <typename T, bool KCONTIG, int R>
__device__ __forceinline__ void load_one(T (&f)[R], const T *X, int ld, int k, int r0)
{
#pragma unroll
    for (int r = 0; r < R; ++r) f[r] = KCONTIG ? X[k + (r0 + r) * ld] : X[r0 + r + k * ld];
}

// acc(i,j) += sum_k opA(row0+i, k) * opB(k, col0+j), k ascending, one FMA each.
template <typename T, bool TA, bool TB, int MR, int NR, bool VEC, int UNR, typename ACC>
__device__ __forceinline__ void fma_tile(ACC &acc, const T *__restrict__ sA,
                                         const T *__restrict__ sB, int lda, int ldb, int K,
                                         int row0, int col0)
{
    // A: tile-contiguous iff TA == false;  B: tile-contiguous iff TB == true
    constexpr int KU = KUnroll<T>::value;
    int k = 0;
    // UNR = 2: two k-blocks in flight (the paper's ping-pang, PAPER.md:181 --
    // the next block's fragments load while this block's FMAs issue); the
    // generator enables it where the doubled fragments fit the register budget.
#pragma unroll UNR
    for (; k + KU <= K; k += KU) {
        T a[KU][MR], b[KU][NR];
        load_frag<T, TA, MR, VEC>(a, sA, lda, k, row0);
        load_frag<T, !TB, NR, VEC>(b, sB, ldb, k, col0);
#pragma unroll
        for (int kk = 0; kk < KU; ++kk) acc.rank1([&](int i) { return a[kk][i]; }, [&](int j) { return b[kk][j]; });
    }
#pragma unroll 1
    for (; k < K; ++k) {
        T a[MR], b[NR];
        load_one<T, TA, MR>(a, sA, lda, k, row0);
        load_one<T, !TB, NR>(b, sB, ldb, k, col0);
        acc.rank1([&](int i) { return a[i]; }, [&](int j) { return b[j]; });
    }
}

// C = alpha*acc + beta*C_in, written once per element, never past the tile.
// Cin: where C_in is read (the staged smem copy, or C itself); same ldc.
// Fused alpha/beta epilogue of one lane's MR x NR tile whose element (i, j)
// is C(row0 + i*rs, col0 + j*cs) (column-major, ldc); C_in is read through
// Cin with the same offsets (the staged smem copy, or C itself), never when
// beta == 0.  VR: rows contiguous (rs == 1) and 16-byte vector accesses
// legal.  Columns are processed in blocks whose C_in values fit ~32
// registers; inside a block every C_in load is issued before the first
// store (a load after a store through a possibly aliasing pointer could not
// be hoisted), so their latencies overlap instead of serialising.
template <typename T, int MR, int NR, bool VR, bool CIN_GLOBAL = false>
__device__ __forceinline__ void epilogue_tile(T (&acc)[MR][NR], T *C, const T *Cin, int ldc, int row0, int rs,
                                              int col0, int cs, T alpha, T beta, bool beta_zero)
{
    constexpr int W = VecOf<T>::W;
    constexpr bool V = VR && (MR % W) == 0;
    constexpr int JB0 = (32 / (int)(sizeof(T) / 4)) / MR;
    constexpr int JB = JB0 < 1 ? 1 : (JB0 > NR ? NR : JB0);
#pragma unroll
    for (int j0 = 0; j0 < NR; j0 += JB) {
        T o[MR][JB];
        if (!beta_zero) {
#pragma unroll
            for (int jj = 0; jj < JB; ++jj) {
                if (j0 + jj >= NR) break;
                const T *ci_p = Cin + (int64_t)(col0 + (j0 + jj) * cs) * ldc + row0;
                if (V) {
#pragma unroll
                    for (int q = 0; q < MR / W; ++q) {
                        T t[W];
                        if (CIN_GLOBAL)
                            ldg_vec_cs<T>(ci_p + q * W, t);
                        else
                            ld_vec<T>(ci_p + q * W, t);
#pragma unroll
                        for (int w = 0; w < W; ++w) o[q * W + w][jj] = t[w];
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < MR; ++i) o[i][jj] = CIN_GLOBAL ? ldg_cs(ci_p + i * rs) : ci_p[i * rs];
                }
            }
#pragma unroll
            for (int jj = 0; jj < JB; ++jj) {
                if (j0 + jj >= NR) break;
#pragma unroll
                for (int i = 0; i < MR; ++i) o[i][jj] = fma_rn(alpha, acc[i][j0 + jj], mul_rn(beta, o[i][jj]));
            }
        } else {
#pragma unroll
            for (int jj = 0; jj < JB; ++jj) {
                if (j0 + jj >= NR) break;
#pragma unroll
                for (int i = 0; i < MR; ++i) o[i][jj] = mul_rn(alpha, acc[i][j0 + jj]);
            }
        }
#pragma unroll
        for (int jj = 0; jj < JB; ++jj) {
            if (j0 + jj >= NR) break;
            T *c = C + (int64_t)(col0 + (j0 + jj) * cs) * ldc + row0;
            if (V) {
#pragma unroll
                for (int q = 0; q < MR / W; ++q) {
                    T t[W];
#pragma unroll
                    for (int w = 0; w < W; ++w) t[w] = o[q * W + w][jj];
                    stg_vec_cs<T>(c + q * W, t);
                }
            } else {
#pragma unroll
                for (int i = 0; i < MR; ++i) stg_cs(c + i * rs, o[i][jj]);
            }
        }
    }
}

template <typename T, int MR, int NR, bool VEC>
__device__ __forceinline__ void epilogue(T (&acc)[MR][NR], T *C, const T *Cin, int ldc, int row0,
                                         int col0, T alpha, T beta, bool beta_zero)
{
    epilogue_tile<T, MR, NR, VEC>(acc, C, Cin, ldc, row0, 1, col0, 1, alpha, beta, beta_zero);
}

// One compute warp running FMA tile class `c` over all groups of this CTA.
template <typename T, bool TA, bool TB, int MR, int NR, bool VEC, int UNR>
__device__ __forceinline__ void fma_class_loop(const IaatKParams &p, const IaatClass &c,
                                               unsigned char *smem, uint64_t *full,
                                               uint64_t *empty, int warp, int lane)
{
    int pl, ti, tj;
    bool tile_ok = true;
    if (c.bm == 0) {
        // linear: lane index -> (problem, tile); lanes vary fastest along the
        // tile-contiguous operand (broadcast on the other)
        const int idx = (warp - c.warp_begin) * 32 + lane;
        pl = idx / c.tiles;  // local problem of this lane
        const int t = idx - pl * c.tiles;
        ti = c.colfast ? t / c.tn : t % c.tm;
        tj = c.colfast ? t % c.tn : t / c.tm;
    } else {
        // blocked: the warp owns a bm x bn block of one problem's tiles, so a
        // half-warp's 16-byte loads cover few distinct rows AND columns
        // (shared-memory wavefronts are per half-warp for 128-bit loads)
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
    const T alpha = (T)p.alpha, beta = (T)p.beta;
    const int64_t sab = p.sA * (int64_t)sizeof(T), sbb = p.sB * (int64_t)sizeof(T);
    const int64_t scb = p.sC * (int64_t)sizeof(T);
    int it = 0;
    for (int64_t g = blockIdx.x; g < p.ngroups; g += gridDim.x, ++it) {
        const int s = it % p.S;
        const int64_t b0 = g * p.P;
        const int np = (int)min((int64_t)p.P, p.batch - b0);
        const bool active = tile_ok && pl < np;
        // A tile-contiguous iff !TA, B tile-contiguous iff TB (see load_frag).
        // TN with scalar loads (no 16-byte vectors): each a(i) is its own LDS,
        // so the loads can land in register pairs along i -> FFMA2 as well
        RegTile<T, MR, NR, PairOf<T, !TA || (!VEC && !TB), TB, MR, NR>::value> acc;
        acc.zero();
        mbar_wait(&full[s], (it / p.S) & 1);
        if (active) {
            StageView sv = stage_view(p, smem, s);
            const char *a_first = prob_ptr(p.A, p.Aarr, sab, b0);
            const char *b_first = prob_ptr(p.B, p.Barr, sbb, b0);
            const char *a_prob = p.modeA == IAAT_STAGE_SLAB ? a_first : prob_ptr(p.A, p.Aarr, sab, b0 + pl);
            const char *b_prob = p.modeB == IAAT_STAGE_SLAB ? b_first : prob_ptr(p.B, p.Barr, sbb, b0 + pl);
            const T *sA = reinterpret_cast<const T *>(
                sv.a + smem_offset(p.modeA, a_first, a_prob, sab, p.slotA, pl));
            const T *sB = reinterpret_cast<const T *>(
                sv.b + smem_offset(p.modeB, b_first, b_prob, sbb, p.slotB, pl));
            fma_tile<T, TA, TB, MR, NR, VEC, UNR>(acc, sA, sB, p.lda, p.ldb, p.K, row0, col0);
        }
        if (!p.c_in_smem) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);  // stage s no longer read by this warp
        }
        if (active) {
            const char *c_first = prob_ptr(p.C, cptrs(p), scb, b0);
            const char *c_prob = prob_ptr(p.C, cptrs(p), scb, b0 + pl);
            T *C = const_cast<T *>(reinterpret_cast<const T *>(c_prob));
            const T *Cin = C;
            if (p.c_in_smem) {
                StageView sv = stage_view(p, smem, s);
                Cin = reinterpret_cast<const T *>(
                    sv.c + smem_offset(p.modeC, c_first, c_prob, scb, p.slotC, pl));
            }
            T accv[MR][NR];
            acc.get(accv);
            epilogue<T, MR, NR, VEC>(accv, C, Cin, p.ldc, row0, col0, alpha, beta, p.beta_zero != 0);
        }
        if (p.c_in_smem) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);  // stage s (incl. C_in) no longer read
        }
    }
}

// ------------------------------------------------------------------ programmatic dependent launch
// The GEMM kernels are launched with programmatic stream serialisation
// (launch_cfg in the generated launchers): the next call's grid may be
// scheduled while this one drains, runs its prologue (mbarrier init), and
// then waits in griddepcontrol.wait until every prerequisite grid has
// completed and its memory is visible -- before touching any global
// memory.  Each grid allows its dependents right after that wait.
__device__ __forceinline__ void pdl_wait_and_release()
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Host side: opt the kernel into IAAT_SMEM_LIMIT bytes of dynamic smem on the
// current device, once per device (a single process may drive several GPUs,
// SURVEY 8.5; the attribute belongs to each device's context).
template <typename Kern>
cudaError_t ensure_smem_attr(Kern kern, unsigned long long &done)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = dev < 64 ? 1ull << dev : 0ull;
    if (bit && (__atomic_load_n(&done, __ATOMIC_ACQUIRE) & bit)) return cudaSuccess;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, IAAT_SMEM_LIMIT);
    if (e == cudaSuccess && bit) __atomic_fetch_or(&done, bit, __ATOMIC_RELEASE);
    return e;
}

// Host side: launch with programmatic stream serialisation (off when the
// environment sets IAAT_NO_PDL, for A/B measurement; api.cu).
bool pdl_enabled();

template <typename... Args, typename... Act>
cudaError_t launch_cfg(void (*kern)(Args...), int grid, int block, int smem, cudaStream_t s, Act &&...args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<Act &&>(args)...);
}

// ------------------------------------------------------------------ kernel body
// Dispatcher: generated by gen/generate.py (the install-time stage); its
// static run() switches on the catalog code of the warp's class.
template <typename T, typename Dispatcher>
__device__ __forceinline__ void pipeline_kernel_body(const IaatKParams &p)
{
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + IAAT_MAX_STAGES;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < p.S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], p.n_compute_warps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    pdl_wait_and_release();
    if (warp == p.n_compute_warps) {
        producer_loop<T>(p, smem, full, empty, lane);
        return;
    }
    int c = 0;
#pragma unroll
    for (int q = 1; q < IAAT_MAX_CLASSES; ++q)
        if (q < p.nclasses && warp >= p.cls[q].warp_begin) c = q;
    Dispatcher::run(p, p.cls[c], smem, full, empty, warp, lane);
}

// ------------------------------------------------------------------ quick-return path
// alpha == 0 or K == 0 (and beta != 1): C = beta*C, or C = 0 without reading
// C when beta == 0 (readings A3-A5).  A and B are never read.
template <typename T>
__global__ void scale_kernel(char *C, void *const *Carr, int64_t sC, int M, int N, int ldc,
                             int64_t batch, double beta_d)
{
    const T beta = (T)beta_d;
    const int64_t per = (int64_t)M * N;
    const int64_t total = per * batch;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = x / per;
        const int64_t e = x - b * per;
        const int j = (int)(e / M), i = (int)(e - (int64_t)j * M);
        T *c = Carr ? reinterpret_cast<T *>(Carr[b]) : reinterpret_cast<T *>(C + b * sC * (int64_t)sizeof(T));
        T *q = c + i + (int64_t)j * ldc;
        *q = beta == (T)0 ? (T)0 : mul_rn(beta, *q);
    }
}

}  // namespace iaat
