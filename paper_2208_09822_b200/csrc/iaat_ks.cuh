// iaat_ks.cuh -- the K-streamed ("ks") kernel family: TMA tensor-map staging
// of K-chunks, for the mid/large end of the small-GEMM domain.
//
// The slab family (iaat_device.cuh) stages whole problems in their global
// layout.  Past ~n = 36 that pins whole problems in shared memory while
// they are computed (n = 80 fp32: 77 KB per problem with C_in), leaves few
// warps per SM, and reads operands that are contiguous along k with bank
// conflicts whenever ld * elt is a multiple of 128 B.  Here a unit of P
// consecutive problems is streamed through an S-stage ring in K-chunks of
// kc = 128 B / elt (32 fp32, 16 fp64) with ONE 3-D TMA box per operand per
// chunk (coordinates {k or row, col or k, problem}), straight from the
// caller's layout -- still no pack pass: the copy
// engine places each chunk in shared memory as it lies in HBM, with the
// 128-byte swizzle for operands that are contiguous along k so that the
// compute warps read them conflict-free.  Accumulators stay in registers
// across the chunks of a unit; alpha/beta are fused in the epilogue and C_in
// is read from global (the producer prefetches it into L2 at unit start).
//
// Smem layouts of one stage (per operand, P problems):
//   MN-major (op(A) = A with A stored M x K; op(B) = B^T with B stored N x K):
//       box {pitch, kc, P} -> [P][kc][pitch]   (pitch >= D, elements)
//   K-major  (op(A) = A^T; op(B) = B):
//       box {kc, D, P}     -> [P][D][kc], 128 B rows, SWIZZLE_128B:
//       16-byte chunk q of row r lives at chunk q ^ (r & 7).
// Tile -> element maps (exact tiles; no predicated edge code):
//   MN-major dim: tile t covers base + t*R + {0..R-1}  (vector loads along it)
//   K-major dim:  tile t covers base + t + nt*{0..R-1} (interleaved, so that
//                 neighbouring lanes read neighbouring rows -> distinct
//                 swizzle chunks -> one wavefront per half-warp)
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "iaat_device.cuh"
#include "iaat_params.h"

namespace iaat {

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2,
                                            uint64_t *bar, uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map)
{
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// First stage of the ring: the first 1024 B boundary after the mbarriers
// (SWIZZLE_128B boxes need 1024 B-aligned destinations; the dynamic smem
// base itself is only guaranteed 16 B alignment).  The plan reserves
// IAAT_KS_BAR_BYTES + 1024 B in front of the ring.
__device__ __forceinline__ unsigned char *ks_ring(unsigned char *smem)
{
    const uint32_t b = smem_u32(smem);
    const uint32_t r = (b + IAAT_KS_BAR_BYTES + 1023u) & ~1023u;
    return smem + (r - b);
}

// ------------------------------------------------------------------ producer
// One warp, lane 0 issues.  Stage s of the ring = [A box | B box] of chunk c
// of unit u; full[s] completes when both boxes have landed (tx bytes = the
// full box sizes, out-of-bounds elements of a ragged last chunk or unit are
// zero-filled by the copy engine and never used by the compute warps).
template <typename T, bool TA, bool TB>
__device__ void ks_producer(const IaatKsParams &p, const CUtensorMap *tmA, const CUtensorMap *tmB,
                            unsigned char *smem, uint64_t *full, uint64_t *empty, int lane)
{
    if (lane != 0) return;
    prefetch_tmap(tmA);
    prefetch_tmap(tmB);
    const uint64_t pol = policy_evict_first();
    const uint32_t tx = (uint32_t)(p.a_tx + p.b_tx);
    unsigned char *ring = ks_ring(smem);
    int it = 0;
    for (int64_t u = blockIdx.x; u < p.nunits; u += gridDim.x) {
        const int b0 = (int)(u * p.P);
        if (!p.beta_zero) {
            // C_in of the unit's problems is read by the epilogue: warm L2 now
            const int np = (int)min((int64_t)p.P, p.batch - b0);
            const int64_t scb = p.sC * (int64_t)sizeof(T);
            const char *first = p.C + (int64_t)b0 * scb;
            const int64_t span = (int64_t)(np - 1) * scb + ((int64_t)(p.N - 1) * p.ldc + p.M) * (int64_t)sizeof(T);
            uintptr_t lo = reinterpret_cast<uintptr_t>(first) & ~(uintptr_t)15;
            uintptr_t hi = (reinterpret_cast<uintptr_t>(first) + (uintptr_t)span + 15) & ~(uintptr_t)15;
            bulk_prefetch_l2(reinterpret_cast<const void *>(lo), (uint32_t)(hi - lo));
        }
        for (int c = 0; c < p.nchunks; ++c, ++it) {
            const int s = it % p.S;
            if (it >= p.S) mbar_wait(&empty[s], ((it / p.S) - 1) & 1);
            unsigned char *st = ring + (size_t)s * p.stage_bytes;
            mbar_arrive_expect_tx(&full[s], tx);
            const int k0 = c * p.kc;
            if (TA) tma_load_3d(st, tmA, k0, 0, b0, &full[s], pol);                 // A: K x M, K-major
            else    tma_load_3d(st, tmA, 0, k0, b0, &full[s], pol);                 // A: M x K, MN-major
            if (TB) tma_load_3d(st + p.a_bytes, tmB, 0, k0, b0, &full[s], pol);     // B: N x K, MN-major
            else    tma_load_3d(st + p.a_bytes, tmB, k0, 0, b0, &full[s], pol);     // B: K x N, K-major
        }
    }
}

// ------------------------------------------------------------------ operand readers
// K-major swizzled operand: byte offset of row r's 16-byte chunk q is
// (r * 128) | ((q ^ (r & 7)) << 4) == ((r * 128) | ((r & 7) << 4)) ^ (q << 4).
__device__ __forceinline__ uint32_t kmaj_row_base(int r_abs) { return ((uint32_t)r_abs << 7) | ((uint32_t)(r_abs & 7) << 4); }

// One k-block (KU = 16 B / elt k-steps) of R elements along the tile dim.
// f[kk][r]: operand value at (tile element r, k = kb + kk).
template <typename T, bool KMAJ, int R, int NB>
__device__ __forceinline__ void ks_load_block(T (&f)[16 / sizeof(T)][R], const unsigned char *st,
                                              const uint32_t (&rb)[NB], uint32_t mn_off, int pitch_bytes,
                                              int kb)
{
    constexpr int KU = 16 / sizeof(T);
    if (KMAJ) {
        const uint32_t q = (uint32_t)(kb / KU) << 4;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            T t[KU];
            ld_vec<T>(reinterpret_cast<const T *>(st + (rb[r < NB ? r : 0] ^ q)), t);
#pragma unroll
            for (int kk = 0; kk < KU; ++kk) f[kk][r] = t[kk];
        }
    } else {
        constexpr int W = 16 / sizeof(T);
#pragma unroll
        for (int kk = 0; kk < KU; ++kk) {
            const T *row = reinterpret_cast<const T *>(st + mn_off + (uint32_t)((kb + kk) * pitch_bytes));
            if ((R % W) == 0) {
#pragma unroll
                for (int v = 0; v < R / W; ++v) ld_vec<T>(row + v * W, &f[kk][v * W]);
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) f[kk][r] = row[r];
            }
        }
    }
}

// Single k-step (scalar) for a ragged chunk tail.
template <typename T, bool KMAJ, int R, int NB>
__device__ __forceinline__ void ks_load_one(T (&f)[R], const unsigned char *st, const uint32_t (&rb)[NB],
                                            uint32_t mn_off, int pitch_bytes, int k)
{
    constexpr int KU = 16 / sizeof(T);
    if (KMAJ) {
        const uint32_t q = (uint32_t)(k / KU) << 4, w = (uint32_t)(k % KU) * sizeof(T);
#pragma unroll
        for (int r = 0; r < R; ++r) f[r] = *reinterpret_cast<const T *>(st + ((rb[r < NB ? r : 0] ^ q) + w));
    } else {
        const T *row = reinterpret_cast<const T *>(st + mn_off + (uint32_t)(k * pitch_bytes));
#pragma unroll
        for (int r = 0; r < R; ++r) f[r] = row[r];
    }
}

// ------------------------------------------------------------------ FMA class (per-thread tile)
template <typename T, bool TA, bool TB, int MR, int NR, int UNR>
__device__ __forceinline__ void ks_fma_class_loop(const IaatKsParams &p, const IaatClass &c, unsigned char *smem,
                                                  uint64_t *full, uint64_t *empty, int warp, int lane)
{
    constexpr int KU = 16 / sizeof(T);
    constexpr bool AK = TA;   // op(A) K-major in smem
    constexpr bool BK = !TB;  // op(B) K-major in smem
    // lane -> (local problem, tile row, tile col)
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
    if (!tile_ok) {
        ti = 0;
        tj = 0;
    }
    // first element of the lane's tile along each dim (exact tiles; see the
    // header comment for the MN-major / K-major element maps)
    const int row0 = AK ? c.row_base + ti : c.row_base + ti * MR;
    const int col0 = BK ? c.col_base + tj : c.col_base + tj * NR;
    // smem addressing inside a stage (problem pl of the unit)
    const int pc = min(pl, p.P - 1);
    uint32_t ra[AK ? MR : 1], rbB[BK ? NR : 1];
#pragma unroll
    for (int i = 0; i < (AK ? MR : 1); ++i) ra[i] = kmaj_row_base(pc * p.M + row0 + c.tm * i);
#pragma unroll
    for (int j = 0; j < (BK ? NR : 1); ++j) rbB[j] = kmaj_row_base(pc * p.N + col0 + c.tn * j);
    const uint32_t a_mn = AK ? 0u : (uint32_t)((pc * p.kc * p.a_pitch + row0) * (int)sizeof(T));
    const uint32_t b_mn = BK ? 0u : (uint32_t)((pc * p.kc * p.b_pitch + col0) * (int)sizeof(T));
    const int a_pb = p.a_pitch * (int)sizeof(T), b_pb = p.b_pitch * (int)sizeof(T);
    const T alpha = (T)p.alpha, beta = (T)p.beta;
    const int64_t scb = p.sC * (int64_t)sizeof(T);
    const unsigned char *ring = ks_ring(smem);

    int it = 0;
    for (int64_t u = blockIdx.x; u < p.nunits; u += gridDim.x) {
        const int64_t b0 = u * p.P;
        const bool active = tile_ok && (b0 + pl) < p.batch && pl < p.P;
        T acc[MR][NR];
#pragma unroll
        for (int i = 0; i < MR; ++i)
#pragma unroll
            for (int j = 0; j < NR; ++j) acc[i][j] = (T)0;
        for (int ch = 0; ch < p.nchunks; ++ch, ++it) {
            const int s = it % p.S;
            mbar_wait(&full[s], (it / p.S) & 1);
            if (active) {
                const unsigned char *st = ring + (size_t)s * p.stage_bytes;
                const unsigned char *sa = st, *sb = st + p.a_bytes;
                const int kv = min(p.kc, p.K - ch * p.kc);
                int kb = 0;
#pragma unroll UNR
                for (; kb + KU <= kv; kb += KU) {
                    T a[KU][MR], b[KU][NR];
                    ks_load_block<T, AK, MR>(a, sa, ra, a_mn, a_pb, kb);
                    ks_load_block<T, BK, NR>(b, sb, rbB, b_mn, b_pb, kb);
#pragma unroll
                    for (int kk = 0; kk < KU; ++kk)
#pragma unroll
                        for (int j = 0; j < NR; ++j)
#pragma unroll
                            for (int i = 0; i < MR; ++i) acc[i][j] = fma_rn(a[kk][i], b[kk][j], acc[i][j]);
                }
#pragma unroll 1
                for (; kb < kv; ++kb) {
                    T a[MR], b[NR];
                    ks_load_one<T, AK, MR>(a, sa, ra, a_mn, a_pb, kb);
                    ks_load_one<T, BK, NR>(b, sb, rbB, b_mn, b_pb, kb);
#pragma unroll
                    for (int j = 0; j < NR; ++j)
#pragma unroll
                        for (int i = 0; i < MR; ++i) acc[i][j] = fma_rn(a[i], b[j], acc[i][j]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (active) {
            // fused epilogue: C = alpha*acc + beta*C_in (C_in never read when beta == 0)
            T *C = reinterpret_cast<T *>(p.C + (b0 + pl) * scb);
            constexpr int W = 16 / sizeof(T);
#pragma unroll
            for (int j = 0; j < NR; ++j) {
                const int col = BK ? col0 + c.tn * j : col0 + j;
                T *cc = C + (int64_t)col * p.ldc;
                if (!AK && (MR % W) == 0 && p.c_vec) {
#pragma unroll
                    for (int v = 0; v < MR / W; ++v) {
                        T o[W];
                        if (p.beta_zero) {
#pragma unroll
                            for (int w = 0; w < W; ++w) o[w] = mul_rn(alpha, acc[v * W + w][j]);
                        } else {
                            T ci[W];
                            ld_vec<T>(cc + row0 + v * W, ci);
#pragma unroll
                            for (int w = 0; w < W; ++w) o[w] = fma_rn(alpha, acc[v * W + w][j], mul_rn(beta, ci[w]));
                        }
                        st_vec<T>(cc + row0 + v * W, o);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < MR; ++i) {
                        T *q = cc + (AK ? row0 + c.tm * i : row0 + i);
                        *q = p.beta_zero ? mul_rn(alpha, acc[i][j]) : fma_rn(alpha, acc[i][j], mul_rn(beta, *q));
                    }
                }
            }
        }
    }
}

// ------------------------------------------------------------------ kernel body
template <typename T, bool TA, bool TB, typename Dispatcher>
__device__ __forceinline__ void ks_kernel_body(const CUtensorMap *tmA, const CUtensorMap *tmB,
                                               const IaatKsParams &p)
{
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + IAAT_KS_MAX_STAGES;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < p.S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], p.n_compute_warps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == p.n_compute_warps) {
        ks_producer<T, TA, TB>(p, tmA, tmB, smem, full, empty, lane);
        return;
    }
    int c = 0;
#pragma unroll
    for (int q = 1; q < IAAT_MAX_CLASSES; ++q)
        if (q < p.nclasses && warp >= p.cls[q].warp_begin) c = q;
    Dispatcher::run(p, p.cls[c], smem, full, empty, warp, lane);
}

}  // namespace iaat
