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

// Measurement-only timing modes (IAAT_DEBUG_KS): compiled
// only into experiment builds (-DIAAT_EXPERIMENTS); the shipped library has
// none of them, so no environment setting can make it skip work.
#ifdef IAAT_EXPERIMENTS
#define IAAT_KS_DEBUG(p) ((p).debug)
#else
#define IAAT_KS_DEBUG(p) 0
#endif

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

// ------------------------------------------------------------------ LDGSTS producer
// Misaligned inputs (odd ld, element-aligned bases): the whole producer warp
// copies each chunk element by element with cp.async (4 or 8 bytes, any
// element alignment) from the caller's layout into the same stage layout the
// TMA boxes produce (MN-major [P][kc][pitch] / K-major [P][D][kc] swizzled),
// lanes walking the contiguous global dimension (coalesced).  Completion:
// each lane's cp.async.mbarrier.arrive.noinc on full[s] (count 32).  Only
// valid elements are copied; the compute warps never read past them.
__device__ __forceinline__ void cp_async_elem(void *dst, const void *src, int bytes)
{
    if (bytes == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async_arrive(uint64_t *bar)
{
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// One operand's chunk [k0, k0 + kv) of problem p (global index b) into its stage region.
//   KMAJ: element (row r < D, k) lives at X[b*sX + r*ld + k]   -> swizzled [p*D + r][k - k0]
//         lanes walk k (one row per warp instruction: coalesced, no division)
//   else: element (row r < D, k) lives at X[b*sX + k*ld + r]   -> [p][k - k0][pitch]
//         lanes walk r along each column
template <typename T, bool KMAJ>
__device__ __forceinline__ void ldgsts_chunk(unsigned char *region, const char *X, int64_t sX, int ld, int D,
                                             int pitch, int kc, int p, int64_t b, int k0, int kv, int lane)
{
    constexpr int KU = 16 / (int)sizeof(T);
    const T *src = reinterpret_cast<const T *>(X) + b * sX;
    if (KMAJ) {
        if (lane < kv) {
            const uint32_t q = (uint32_t)(lane / KU), w = (uint32_t)(lane % KU) * sizeof(T);
            const T *g = src + k0 + lane;
            for (int r = 0; r < D; ++r, g += ld) {
                const int ra = p * D + r;
                const uint32_t off = (((uint32_t)ra << 7) | ((q ^ (uint32_t)(ra & 7)) << 4)) + w;
                cp_async_elem(region + off, g, (int)sizeof(T));
            }
        }
    } else {
        for (int kk = 0; kk < kv; ++kk) {
            const T *g = src + (int64_t)(k0 + kk) * ld;
            unsigned char *d = region + (uint32_t)((p * kc + kk) * pitch) * sizeof(T);
            for (int r = lane; r < D; r += 32) cp_async_elem(d + r * sizeof(T), g + r, (int)sizeof(T));
        }
    }
}

template <typename T, bool TA, bool TB>
__device__ void ks_producer_ldgsts(const IaatKsParams &p, unsigned char *smem, uint64_t *full, uint64_t *empty,
                                   int lane)
{
    constexpr bool AK = TA, BK = !TB;
    unsigned char *ring = ks_ring(smem);
    int s = 0, it = 0;
    uint32_t phase = 0;
    for (int64_t u = blockIdx.x; u < p.nunits; u += gridDim.x) {
        const int64_t b0 = u * p.P;
        const int np = (int)min((int64_t)p.P, p.batch - b0);
        if (!p.beta_zero && lane == 0) {
            const int64_t scb = p.sC * (int64_t)sizeof(T);
            const char *first = p.C + b0 * scb;
            const int64_t span = (int64_t)(np - 1) * scb + ((int64_t)(p.N - 1) * p.ldc + p.M) * (int64_t)sizeof(T);
            uintptr_t lo = reinterpret_cast<uintptr_t>(first) & ~(uintptr_t)15;
            uintptr_t hi = (reinterpret_cast<uintptr_t>(first) + (uintptr_t)span + 15) & ~(uintptr_t)15;
            bulk_prefetch_l2(reinterpret_cast<const void *>(lo), (uint32_t)(hi - lo));
        }
        for (int c = 0; c < p.nchunks; ++c, ++it) {
            if (it >= p.S) mbar_wait(&empty[s], phase);
            unsigned char *st = ring + (size_t)s * p.stage_bytes;
            const int k0 = c * p.kc, kv = min(p.kc, p.K - k0);
            for (int q = 0; q < np; ++q) {
                ldgsts_chunk<T, AK>(st, p.A, p.sA, p.lda, p.M, p.a_pitch, p.kc, q, b0 + q, k0, kv, lane);
                ldgsts_chunk<T, BK>(st + p.a_bytes, p.B, p.sB, p.ldb, p.N, p.b_pitch, p.kc, q, b0 + q, k0, kv, lane);
            }
            cp_async_arrive(&full[s]);
            if (++s == p.S) {
                s = 0;
                if (it >= 2 * p.S - 1) phase ^= 1u;
            }
        }
    }
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
    // K-major boxes (one kc-wide piece of each column) share a 32-byte
    // sector with the column's next chunk: normal L2 priority keeps it
    // (iaat_ksg.cuh ksg_producer, measured there)
    uint64_t pol_norm;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_norm));
    const uint64_t polA = TA ? pol_norm : pol, polB = TB ? pol : pol_norm;
    const uint32_t tx = (uint32_t)(p.a_tx + p.b_tx);
    unsigned char *ring = ks_ring(smem);
    int s = 0, it = 0;
    uint32_t phase = 0;  // parity of the empty barrier to wait for
    for (int64_t u = blockIdx.x; u < p.nunits; u += gridDim.x) {
        const int b0 = (int)(u * p.P);
        if (!p.beta_zero) {
            // C_in of the unit's problems is read by the epilogue: warm L2 now
            const int np = (int)min((int64_t)p.P, p.batch - b0);
            const int64_t scb = p.sC * (int64_t)p.c_elt;
            const char *first = p.C + (int64_t)b0 * scb;
            const int64_t span = (int64_t)(np - 1) * scb + ((int64_t)(p.N - 1) * p.ldc + p.M) * (int64_t)p.c_elt;
            uintptr_t lo = reinterpret_cast<uintptr_t>(first) & ~(uintptr_t)15;
            uintptr_t hi = (reinterpret_cast<uintptr_t>(first) + (uintptr_t)span + 15) & ~(uintptr_t)15;
            bulk_prefetch_l2(reinterpret_cast<const void *>(lo), (uint32_t)(hi - lo));
        }
        for (int c = 0; c < p.nchunks; ++c, ++it) {
#ifdef IAAT_EXPERIMENTS
            if (it >= p.S && (p.debug & 4)) return;  // timing mode: fill the ring once, never refill
#endif
            if (it >= p.S) mbar_wait(&empty[s], phase);
            unsigned char *st = ring + (size_t)s * p.stage_bytes;
            mbar_arrive_expect_tx(&full[s], tx);
            const int k0 = c * p.kc;
            const int kr = p.cplx ? 2 * k0 : k0;  // complex: K-major boxes index the real (re, im) view
            if (TA) tma_load_3d(st, tmA, kr, 0, b0, &full[s], polA);                 // A: K x M, K-major
            else    tma_load_3d(st, tmA, 0, k0, b0, &full[s], polA);                 // A: M x K, MN-major
            if (TB) tma_load_3d(st + p.a_bytes, tmB, 0, k0, b0, &full[s], polB);     // B: N x K, MN-major
            else    tma_load_3d(st + p.a_bytes, tmB, kr, 0, b0, &full[s], polB);     // B: K x N, K-major
            if (++s == p.S) {
                s = 0;
                if (it >= 2 * p.S - 1) phase ^= 1u;  // lap L >= 1 waits for parity (L - 1) & 1
            }
        }
    }
}

// ------------------------------------------------------------------ operand readers
// K-major swizzled operand: byte offset of row r's 16-byte chunk q is
// (r * 128) | ((q ^ (r & 7)) << 4) == ((r * 128) | ((r & 7) << 4)) ^ (q << 4).
__device__ __forceinline__ uint32_t kmaj_row_base(int r_abs) { return ((uint32_t)r_abs << 7) | ((uint32_t)(r_abs & 7) << 4); }

// One k-step of an MN-major operand: R consecutive elements at byte offset
// `off` of the stage region (16-byte vectors when R allows).
template <typename T, int R>
__device__ __forceinline__ void ks_load_mn(T (&f)[R], const unsigned char *st, uint32_t off)
{
    constexpr int W = 16 / sizeof(T);
    const T *row = reinterpret_cast<const T *>(st + off);
    if ((R % W) == 0) {
#pragma unroll
        for (int v = 0; v < R / W; ++v) ld_vec<T>(row + v * W, &f[v * W]);
    } else {
#pragma unroll
        for (int r = 0; r < R; ++r) f[r] = row[r];
    }
}

// ------------------------------------------------------------------ FMA k-block fragments
// Fragments of one k-block (KU k-steps) of a lane's tile: K-major operands
// for all KU k-steps (one 16-byte load per row / column), MN-major operands
// for the block's first k-step only (the remaining KU-1 are loaded inside
// ks_frag_fma, one k-step ahead of their FMAs).
template <typename T, bool AK, bool BK, int MR, int NR>
struct KsFrag {
    static constexpr int KU = 16 / sizeof(T);
    T ka[AK ? KU : 1][MR];
    T kb[BK ? KU : 1][NR];
    T ma[AK ? 1 : MR];
    T mb[BK ? 1 : NR];
};

// Shared-memory addressing of one operand inside the current stage, as byte
// offsets from the dynamic smem base.
//   K-major (swizzled rows): element (r-th row of the lane, k) lives at
//       (base[r] ^ ((k / KU) << 4)) + (k % KU) * elt,  base[r] = stage + row_r*128 | (row_r & 7) << 4
//     UNI: every row of the lane has the same swizzle phase (row stride a
//       multiple of 8), so one XOR serves all rows: (base[0] ^ q) + r * rstride.
//   MN-major: element (tile element r, k) at mn + k * pitch + r * elt.
template <bool KMAJ, bool UNI, int R>
struct KsOpnd {
    uint32_t base[KMAJ && !UNI ? R : 1];
    uint32_t rstride;  // UNI: byte stride between the lane's rows
    uint32_t pitch;    // MN-major: bytes per k-step
};

template <typename T, bool KMAJ, bool UNI, int R>
__device__ __forceinline__ void ks_ld_kblock(T (&f)[16 / sizeof(T)][R], const unsigned char *smem,
                                             const KsOpnd<KMAJ, UNI, R> &o, int kb)
{
    constexpr int KU = 16 / sizeof(T);
    const uint32_t q = (uint32_t)(kb / KU) << 4;
    const uint32_t x0 = o.base[0] ^ q;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        T t[KU];
        const uint32_t off = UNI ? x0 + (uint32_t)r * o.rstride : (o.base[UNI ? 0 : r] ^ q);
        ld_vec<T>(reinterpret_cast<const T *>(smem + off), t);
#pragma unroll
        for (int kk = 0; kk < KU; ++kk) f[kk][r] = t[kk];
    }
}

template <typename T, bool AK, bool BK, bool UA, bool UB, int MR, int NR>
__device__ __forceinline__ void ks_frag_load(KsFrag<T, AK, BK, MR, NR> &f, const unsigned char *smem,
                                             const KsOpnd<AK, UA, MR> &oa, const KsOpnd<BK, UB, NR> &ob,
                                             uint32_t a_mn, uint32_t b_mn, int kb)
{
    constexpr int KU = 16 / sizeof(T);
    if (AK) ks_ld_kblock<T, AK, UA, MR>(reinterpret_cast<T (&)[KU][MR]>(f.ka), smem, oa, kb);
    else ks_load_mn<T, MR>(reinterpret_cast<T (&)[MR]>(f.ma), smem, a_mn + (uint32_t)kb * oa.pitch);
    if (BK) ks_ld_kblock<T, BK, UB, NR>(reinterpret_cast<T (&)[KU][NR]>(f.kb), smem, ob, kb);
    else ks_load_mn<T, NR>(reinterpret_cast<T (&)[NR]>(f.mb), smem, b_mn + (uint32_t)kb * ob.pitch);
}

// acc(i,j) += sum over the KU k-steps of the block, k ascending, one FMA each.
template <typename T, bool AK, bool BK, bool UA, bool UB, int MR, int NR, typename ACC>
__device__ __forceinline__ void ks_frag_fma(ACC &acc, const KsFrag<T, AK, BK, MR, NR> &f,
                                            const unsigned char *smem, const KsOpnd<AK, UA, MR> &oa,
                                            const KsOpnd<BK, UB, NR> &ob, uint32_t a_mn, uint32_t b_mn, int kb)
{
    constexpr int KU = 16 / sizeof(T);
    T ma[2][AK ? 1 : MR], mb[2][BK ? 1 : NR];
    const uint32_t a0 = a_mn + (uint32_t)kb * oa.pitch, b0 = b_mn + (uint32_t)kb * ob.pitch;
#pragma unroll
    for (int kk = 0; kk < KU; ++kk) {
        if (kk + 1 < KU) {  // next k-step of the MN-major operands
            if (!AK) ks_load_mn<T, MR>(reinterpret_cast<T (&)[MR]>(ma[(kk + 1) & 1]), smem,
                                       a0 + (uint32_t)(kk + 1) * oa.pitch);
            if (!BK) ks_load_mn<T, NR>(reinterpret_cast<T (&)[NR]>(mb[(kk + 1) & 1]), smem,
                                       b0 + (uint32_t)(kk + 1) * ob.pitch);
        }
        acc.rank1(
            [&](int i) { return AK ? f.ka[AK ? kk : 0][i] : (kk == 0 ? f.ma[AK ? 0 : i] : ma[kk & 1][AK ? 0 : i]); },
            [&](int j) { return BK ? f.kb[BK ? kk : 0][j] : (kk == 0 ? f.mb[BK ? 0 : j] : mb[kk & 1][BK ? 0 : j]); });
    }
}

// One K-chunk (kv valid k-steps) of the lane's tile.  sa / sb: byte offsets
// of the stage's A / B regions from the smem base; ra / rb: the lane's
// swizzled row / column bases inside a region (K-major operands), a_mn /
// b_mn: the lane's first element inside a region (MN-major operands).
template <typename T, bool AK, bool BK, bool UA, bool UB, int MR, int NR, int UNR, int NA, int NB, typename ACC>
__device__ __forceinline__ void ks_chunk(ACC &acc, const unsigned char *smem, uint32_t sa, uint32_t sb,
                                         const uint32_t (&ra)[NA], const uint32_t (&rb)[NB], uint32_t a_mn,
                                         uint32_t b_mn, uint32_t a_pitch, uint32_t b_pitch, uint32_t a_rs,
                                         uint32_t b_rs, int kv)
{
    constexpr int KU = 16 / sizeof(T);
    KsOpnd<AK, UA, MR> oa;
    KsOpnd<BK, UB, NR> ob;
#pragma unroll
    for (int i = 0; i < (AK && !UA ? MR : 1); ++i) oa.base[i] = sa + ra[i < NA ? i : 0];
#pragma unroll
    for (int j = 0; j < (BK && !UB ? NR : 1); ++j) ob.base[j] = sb + rb[j < NB ? j : 0];
    oa.rstride = a_rs;
    ob.rstride = b_rs;
    oa.pitch = a_pitch;
    ob.pitch = b_pitch;
    const uint32_t am = sa + a_mn, bm = sb + b_mn;
    const int kfull = kv & ~(KU - 1);
    int kb = 0;
    if (UNR >= 2) {
        // register double buffering (the paper's ping-pang):
        // the fragments of k-block kb+KU load while the FMAs of kb issue
        KsFrag<T, AK, BK, MR, NR> f0, f1;
        if (kfull > 0) ks_frag_load<T, AK, BK, UA, UB, MR, NR>(f0, smem, oa, ob, am, bm, 0);
        for (; kb < kfull; kb += 2 * KU) {
            if (kb + KU < kfull) ks_frag_load<T, AK, BK, UA, UB, MR, NR>(f1, smem, oa, ob, am, bm, kb + KU);
            ks_frag_fma<T, AK, BK, UA, UB, MR, NR>(acc, f0, smem, oa, ob, am, bm, kb);
            if (kb + KU >= kfull) {
                kb += KU;
                break;
            }
            if (kb + 2 * KU < kfull) ks_frag_load<T, AK, BK, UA, UB, MR, NR>(f0, smem, oa, ob, am, bm, kb + 2 * KU);
            ks_frag_fma<T, AK, BK, UA, UB, MR, NR>(acc, f1, smem, oa, ob, am, bm, kb + KU);
        }
    } else {
#pragma unroll 2
        for (; kb < kfull; kb += KU) {
            KsFrag<T, AK, BK, MR, NR> f0;
            ks_frag_load<T, AK, BK, UA, UB, MR, NR>(f0, smem, oa, ob, am, bm, kb);
            ks_frag_fma<T, AK, BK, UA, UB, MR, NR>(acc, f0, smem, oa, ob, am, bm, kb);
        }
    }
    // ragged tail of the chunk (K % KU), one k-step at a time
#pragma unroll 1
    for (; kb < kv; ++kb) {
        T a[MR], b[NR];
        const uint32_t q = (uint32_t)(kb / KU) << 4, w = (uint32_t)(kb % KU) * sizeof(T);
#pragma unroll
        for (int i = 0; i < MR; ++i)
            a[i] = AK ? *reinterpret_cast<const T *>(smem + ((UA ? (oa.base[0] ^ q) + i * a_rs : (oa.base[AK && !UA ? i : 0] ^ q)) + w))
                      : *reinterpret_cast<const T *>(smem + am + (uint32_t)kb * a_pitch + i * sizeof(T));
#pragma unroll
        for (int j = 0; j < NR; ++j)
            b[j] = BK ? *reinterpret_cast<const T *>(smem + ((UB ? (ob.base[0] ^ q) + j * b_rs : (ob.base[BK && !UB ? j : 0] ^ q)) + w))
                      : *reinterpret_cast<const T *>(smem + bm + (uint32_t)kb * b_pitch + j * sizeof(T));
        acc.rank1([&](int i) { return a[i]; }, [&](int j) { return b[j]; });
    }
}

// ------------------------------------------------------------------ FMA class (per-thread tile)
// UMODE: 0 = choose the swizzle addressing per call (uniform-phase or
// general code path, both compiled); 1 = uniform-phase only (the planner
// guarantees tm, tn multiples of 8 for the K-major dims); 2 = general only.
// Single paths keep the register footprint of the big tiles down.
template <typename T, bool TA, bool TB, int MR, int NR, int UNR, int UMODE = 0>
__device__ __forceinline__ void ks_fma_class_loop(const IaatKsParams &p, const IaatClass &c, unsigned char *smem,
                                                  uint64_t *full, uint64_t *empty, int warp, int lane)
{
    constexpr int KU = 16 / sizeof(T);
    constexpr bool AK = TA;   // op(A) K-major in smem
    constexpr bool BK = !TB;  // op(B) K-major in smem
    // Parameters are read once into registers: the function is not inlined,
    // p and c arrive as generic pointers, and a load through them after a
    // store to C could not be hoisted by the compiler.
    const int K = p.K, kc = p.kc, nchunks = p.nchunks, P = p.P, S = p.S, M = p.M, N = p.N, ldc = p.ldc;
    const int stage_bytes = p.stage_bytes, a_bytes = p.a_bytes;
    const int dbg = IAAT_KS_DEBUG(p);
    const bool beta_zero = p.beta_zero != 0, c_vec = p.c_vec != 0;
    const int64_t nunits = p.nunits, batch = p.batch;
    char *const Cbase = p.C;
    const int tm = c.tm, tn = c.tn;
    // lane -> (local problem, tile row, tile col)
    int pl, ti, tj;
    bool tile_ok = true;
    if (c.bm == 0) {
        const int idx = (warp - c.warp_begin) * 32 + lane;
        pl = idx / c.tiles;
        const int t = idx - pl * c.tiles;
        ti = c.colfast ? t / tn : t % tm;
        tj = c.colfast ? t % tn : t / tm;
    } else {
        const int bn = 32 / c.bm;
        const int nbm = (tm + c.bm - 1) / c.bm, nbn = (tn + bn - 1) / bn;
        const int wb = warp - c.warp_begin;
        pl = wb / (nbm * nbn);
        const int blk = wb - pl * (nbm * nbn);
        ti = (blk % nbm) * c.bm + lane % c.bm;
        tj = (blk / nbm) * bn + lane / c.bm;
        tile_ok = ti < tm && tj < tn;
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
    const int pc = min(pl, P - 1);
    uint32_t ra[AK ? MR : 1], rbB[BK ? NR : 1];
#pragma unroll
    for (int i = 0; i < (AK ? MR : 1); ++i) ra[i] = kmaj_row_base(pc * M + row0 + tm * i);
#pragma unroll
    for (int j = 0; j < (BK ? NR : 1); ++j) rbB[j] = kmaj_row_base(pc * N + col0 + tn * j);
    const uint32_t a_mn = AK ? 0u : (uint32_t)((pc * kc * p.a_pitch + row0) * (int)sizeof(T));
    const uint32_t b_mn = BK ? 0u : (uint32_t)((pc * kc * p.b_pitch + col0) * (int)sizeof(T));
    const uint32_t a_pb = (uint32_t)(p.a_pitch * (int)sizeof(T)), b_pb = (uint32_t)(p.b_pitch * (int)sizeof(T));
    // uniform swizzle phase across the lane's rows / columns (row stride tm
    // or tn a multiple of 8): one XOR per k-block instead of one per row
    const bool ua = AK && (MR == 1 || (tm & 7) == 0), ub = BK && (NR == 1 || (tn & 7) == 0);
    const uint32_t a_rs = (uint32_t)tm * 128u, b_rs = (uint32_t)tn * 128u;
    const uint32_t ring_off = (uint32_t)(ks_ring(smem) - smem);
    const T alpha = (T)p.alpha, beta = (T)p.beta;
    const int64_t scb = p.sC * (int64_t)sizeof(T);

    int s = 0;
    uint32_t phase = 0;
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int64_t b0 = u * P;
        const bool active = tile_ok && (b0 + pl) < batch && pl < P;
        RegTile<T, MR, NR, PairOf<T, !AK, !BK, MR, NR>::value> acc;
        acc.zero();
        for (int ch = 0; ch < nchunks; ++ch) {
            if (!(dbg & 4)) mbar_wait(&full[s], phase);
            if (active && !(dbg & 1)) {
                const uint32_t sa = ring_off + (uint32_t)(s * stage_bytes), sb = sa + (uint32_t)a_bytes;
                const int kv = min(kc, K - ch * kc);
                // warp-uniform: one code path per swizzle-phase case
                if (UMODE == 1)
                    ks_chunk<T, AK, BK, AK, BK, MR, NR, UNR>(acc, smem, sa, sb, ra, rbB, a_mn, b_mn, a_pb, b_pb,
                                                             a_rs, b_rs, kv);
                else if (UMODE == 2)
                    ks_chunk<T, AK, BK, false, false, MR, NR, UNR>(acc, smem, sa, sb, ra, rbB, a_mn, b_mn, a_pb,
                                                                   b_pb, a_rs, b_rs, kv);
                else if (ua && ub)
                    ks_chunk<T, AK, BK, AK, BK, MR, NR, UNR>(acc, smem, sa, sb, ra, rbB, a_mn, b_mn, a_pb, b_pb,
                                                             a_rs, b_rs, kv);
                else if (ua)
                    ks_chunk<T, AK, BK, AK, false, MR, NR, UNR>(acc, smem, sa, sb, ra, rbB, a_mn, b_mn, a_pb, b_pb,
                                                                a_rs, b_rs, kv);
                else if (ub)
                    ks_chunk<T, AK, BK, false, BK, MR, NR, UNR>(acc, smem, sa, sb, ra, rbB, a_mn, b_mn, a_pb, b_pb,
                                                                a_rs, b_rs, kv);
                else
                    ks_chunk<T, AK, BK, false, false, MR, NR, UNR>(acc, smem, sa, sb, ra, rbB, a_mn, b_mn, a_pb,
                                                                   b_pb, a_rs, b_rs, kv);
            }
            __syncwarp();
            if (lane == 0 && !(dbg & 4)) mbar_arrive(&empty[s]);
            if (++s == S) {
                s = 0;
                phase ^= 1u;
            }
        }
        if (active && !(dbg & 2)) {
            // fused epilogue: C = alpha*acc + beta*C_in (C_in never read when beta == 0)
            T *C = reinterpret_cast<T *>(Cbase + (b0 + pl) * scb);
            T accv[MR][NR];
            acc.get(accv);
            if (!AK && c_vec)
                epilogue_tile<T, MR, NR, true, true>(accv, C, C, ldc, row0, 1, col0, BK ? tn : 1, alpha, beta,
                                                     beta_zero);
            else
                epilogue_tile<T, MR, NR, false, true>(accv, C, C, ldc, row0, AK ? tm : 1, col0, BK ? tn : 1, alpha,
                                                      beta, beta_zero);
        }
    }
}

// ------------------------------------------------------------------ DMMA class (fp64 warp tile)
// One warp owns a (8*WM) x (8*WN) block of one problem's C for the whole
// unit (accumulators in registers across the K-chunks), issued as DMMA.8x8x4
// (mma.sync.m8n8k4.f64, the only FP64 tensor-core instruction on sm_100a) in
// the transposed form D' = op(B)^T op(A)^T of iaat_dmma.cuh, so a lane's two
// accumulators are two consecutive rows of one C column.
// k mapping inside a chunk: DMMA step s (4 per 16-k chunk) gives position t
// the k-value 4s + t (the same for both fragments): MN-major operands are
// then read as 4 consecutive k-rows per half-warp (pitch = 4 mod 16 doubles,
// conflict-free), K-major ones with at most a 2-way bank conflict.
// A ragged last chunk reads the copy engine's zero fill past K (0 * 0 adds
// nothing); no MMA is predicated.
__device__ __forceinline__ void ks_dmma_8x8x4(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// Byte offset (inside a stage region) of element (row r_abs, k) of an fp64
// operand: K-major swizzled 128-byte rows or MN-major rows of `pitch` doubles.
template <bool KMAJ>
__device__ __forceinline__ uint32_t ks_f64_off(int r_abs, int k, int pitch_el, int pk)
{
    if (KMAJ) return (((uint32_t)r_abs << 7) | ((uint32_t)((k >> 1) ^ (r_abs & 7)) << 4)) + (uint32_t)(k & 1) * 8u;
    return (uint32_t)(pk * pitch_el + k * pitch_el + r_abs) * 8u;
}

template <bool TA, bool TB, int WM, int WN>
__device__ __forceinline__ void ks_dmma_class_loop(const IaatKsParams &p, const IaatClass &c, unsigned char *smem,
                                                   uint64_t *full, uint64_t *empty, int warp, int lane)
{
    constexpr bool AK = TA, BK = !TB;
    const int K = p.K, kc = p.kc, nchunks = p.nchunks, P = p.P, S = p.S, M = p.M, N = p.N, ldc = p.ldc;
    const int stage_bytes = p.stage_bytes, a_bytes = p.a_bytes;
    const int dbg = IAAT_KS_DEBUG(p);
    const bool beta_zero = p.beta_zero != 0, c_vec = p.c_vec != 0;
    const int64_t nunits = p.nunits, batch = p.batch;
    const int g = lane >> 2, t = lane & 3;
    const int wi = warp - c.warp_begin;
    const int pl = wi / c.tiles, tt = wi - pl * c.tiles;
    const int ti = c.colfast ? tt / c.tn : tt % c.tm;
    const int tj = c.colfast ? tt % c.tn : tt / c.tm;
    const int row0 = c.row_base + ti * 8 * WM, col0 = c.col_base + tj * 8 * WN;
    const int pc = min(pl, P - 1);
    // per-lane offsets of fragment element k = t (step 0 of a chunk); step s
    // adds 4 k-rows (MN-major) or two 16-byte chunks (K-major, via the XOR)
    // K-major (swizzled) operands: MMA row g reads smem row pi(g) = 2g mod 8
    // (+1 for g >= 4) of its 8-row block.  A quarter-warp (g = 0..3 or 4..7,
    // t = 0..3) then reads rows whose swizzle phases {0,2,4,6} / {1,3,5,7}
    // XOR the chunk pair {2st, 2st+1} into 8 different 16-byte chunks --
    // conflict-free, where g -> row g put two lanes on one bank (ncu round 1:
    // 43 % of the shared wavefronts were conflicts).  The permutation is
    // undone in the epilogue (it only relabels C rows / columns).
    const int gA = AK ? (((2 * g) & 7) | (g >> 2)) : g, gB = BK ? (((2 * g) & 7) | (g >> 2)) : g;
    uint32_t oa[WM], ob[WN];
#pragma unroll
    for (int mi = 0; mi < WM; ++mi)
        oa[mi] = AK ? ks_f64_off<true>(pc * M + row0 + 8 * mi + gA, t, 0, 0)
                    : ks_f64_off<false>(row0 + 8 * mi + g, t, p.a_pitch, pc * kc);
#pragma unroll
    for (int nj = 0; nj < WN; ++nj)
        ob[nj] = BK ? ks_f64_off<true>(pc * N + col0 + 8 * nj + gB, t, 0, 0)
                    : ks_f64_off<false>(col0 + 8 * nj + g, t, p.b_pitch, pc * kc);
    const uint32_t a_step = AK ? 0u : (uint32_t)(4 * p.a_pitch * 8), b_step = BK ? 0u : (uint32_t)(4 * p.b_pitch * 8);
    const double alpha = p.alpha, beta = p.beta;
    const int64_t scb = p.sC * 8;
    const uint32_t ring_off = (uint32_t)(ks_ring(smem) - smem);
    const bool tile_ok = pl < P;

    int s = 0;
    uint32_t phase = 0;
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int64_t b0 = u * P;
        const bool active = tile_ok && (b0 + pl) < batch;
        double acc[WM][WN][2];
#pragma unroll
        for (int mi = 0; mi < WM; ++mi)
#pragma unroll
            for (int nj = 0; nj < WN; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
        for (int ch = 0; ch < nchunks; ++ch) {
            mbar_wait(&full[s], phase);
            if (active && !(dbg & 1)) {
                const unsigned char *sa = smem + ring_off + (uint32_t)(s * stage_bytes);
                const unsigned char *sb = sa + a_bytes;
                const int kv = min(kc, K - ch * kc);
                const int nsteps = (kv + 3) >> 2;
                // 5x5 tiles: 100 accumulator registers leave room for two
                // steps of fragments in flight, not four (spill-free at 168)
#pragma unroll(WM * WN >= 25 ? 2 : 4)
                for (int st = 0; st < nsteps; ++st) {
                    double af[WM], bf[WN];
                    // K-major: k = 4*st + t lives in 16-byte chunk 2*st + t/2 -> XOR (st << 5) on the chunk bits
#pragma unroll
                    for (int mi = 0; mi < WM; ++mi)
                        af[mi] = *reinterpret_cast<const double *>(
                            sa + (AK ? (oa[mi] ^ ((uint32_t)st << 5)) : oa[mi] + (uint32_t)st * a_step));
#pragma unroll
                    for (int nj = 0; nj < WN; ++nj)
                        bf[nj] = *reinterpret_cast<const double *>(
                            sb + (BK ? (ob[nj] ^ ((uint32_t)st << 5)) : ob[nj] + (uint32_t)st * b_step));
#pragma unroll
                    for (int mi = 0; mi < WM; ++mi)
#pragma unroll
                        for (int nj = 0; nj < WN; ++nj) ks_dmma_8x8x4(acc[mi][nj][0], acc[mi][nj][1], bf[nj], af[mi]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == S) {
                s = 0;
                phase ^= 1u;
            }
        }
        if (active && !(dbg & 2)) {
            double *C = reinterpret_cast<double *>(p.C + (b0 + pl) * scb);
            // lane (g, t) holds D'[g][2t], D'[g][2t+1]: C column col0 + 8 nj +
            // gB, C rows row0 + 8 mi + the A-side rows of MMA columns 2t,
            // 2t+1 (pi(2t), pi(2t+1) when A is K-major: not adjacent, so
            // scalar accesses; adjacent otherwise: one 16-byte access)
            const int r0 = AK ? (((4 * t) & 7) | ((2 * t) >> 2)) : 2 * t;
            const int r1 = AK ? (((4 * t + 2) & 7) | ((2 * t + 1) >> 2)) : 2 * t + 1;
            const bool vec = c_vec && !AK;
            // per block row: all C_in loads of the row before its stores
            // (overlapped latencies, bounded registers)
#pragma unroll
            for (int mi = 0; mi < WM; ++mi) {
                double ci[WN][2];
                if (!beta_zero) {
#pragma unroll
                    for (int nj = 0; nj < WN; ++nj) {
                        const double *cp = C + (row0 + 8 * mi) + (int64_t)(col0 + 8 * nj + gB) * ldc;
                        if (vec) {
                            ldg_vec_cs<double>(cp + r0, ci[nj]);
                        } else {
                            ci[nj][0] = ldg_cs(cp + r0);
                            ci[nj][1] = ldg_cs(cp + r1);
                        }
                    }
                }
#pragma unroll
                for (int nj = 0; nj < WN; ++nj) {
                    double o[2];
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        o[h] = beta_zero ? mul_rn(alpha, acc[mi][nj][h])
                                         : fma_rn(alpha, acc[mi][nj][h], mul_rn(beta, ci[nj][h]));
                    double *cp = C + (row0 + 8 * mi) + (int64_t)(col0 + 8 * nj + gB) * ldc;
                    if (vec) {
                        stg_vec_cs<double>(cp + r0, o);
                    } else {
                        stg_cs(cp + r0, o[0]);
                        stg_cs(cp + r1, o[1]);
                    }
                }
            }
        }
    }
}

// ------------------------------------------------------------------ complex DMMA (ZGEMM) warp tile
// ZGEMM on the fp64 tensor cores (SURVEY f1 + the DMMA path): TMA boxes over
// the real view of the interleaved data (an M x K complex matrix = a 2M x K
// real one), kc = 8 complex k-steps per chunk (K-major rows: 8 complex = 128
// bytes, swizzled; MN-major rows: pitch >= 2M doubles, pitch = 8 mod 16).  One
// 16-byte load gives a lane the (re, im) pair of its fragment element; four
// DMMA per 8x8x4 complex block:
//   D'_re += B_re^T A_re^T + (-B_im)^T A_im^T,   D'_im += B_im^T A_re^T + B_re^T A_im^T
// (transposed form of iaat_dmma.cuh: a lane's accumulators are two
// consecutive C rows).  k mapping: DMMA step s (2 per chunk) gives position t
// the k-value 2t + s for both operands -- on the swizzled K-major rows the
// 4 rows of a half-warp then touch two disjoint bank sets.  A ragged last
// chunk reads the copy engine's zero fill past K.
template <bool KMAJ>
__device__ __forceinline__ uint32_t ksz_off(int r_abs, int k, int pitch_r, int pk)
{
    if (KMAJ) return ((uint32_t)r_abs << 7) | ((uint32_t)(k ^ (r_abs & 7)) << 4);
    return (uint32_t)((pk + k) * pitch_r + 2 * r_abs) * 8u;
}

template <bool TA, bool TB, int WM, int WN>
__device__ __forceinline__ void ks_zdmma_class_loop(const IaatKsParams &p, const IaatClass &c, unsigned char *smem,
                                                    uint64_t *full, uint64_t *empty, int warp, int lane)
{
    constexpr bool AK = TA, BK = !TB;
    const int K = p.K, kc = p.kc, nchunks = p.nchunks, P = p.P, S = p.S, M = p.M, N = p.N, ldc = p.ldc;
    const int stage_bytes = p.stage_bytes, a_bytes = p.a_bytes;
    const bool beta_zero = p.beta_zero != 0;
    const int64_t nunits = p.nunits, batch = p.batch;
    const int g = lane >> 2, t = lane & 3;
    const int wi = warp - c.warp_begin;
    const int pl = wi / c.tiles, tt = wi - pl * c.tiles;
    const int ti = c.colfast ? tt / c.tn : tt % c.tm;
    const int tj = c.colfast ? tt % c.tn : tt / c.tm;
    const int row0 = c.row_base + ti * 8 * WM, col0 = c.col_base + tj * 8 * WN;
    const int pc = min(pl, P - 1);
    uint32_t oa[2][WM], ob[2][WN];  // [step s][block]: element k = 2t + s
#pragma unroll
    for (int st = 0; st < 2; ++st) {
#pragma unroll
        for (int mi = 0; mi < WM; ++mi)
            oa[st][mi] = AK ? ksz_off<true>(pc * M + row0 + 8 * mi + g, 2 * t + st, 0, 0)
                            : ksz_off<false>(row0 + 8 * mi + g, 2 * t + st, p.a_pitch, pc * kc);
#pragma unroll
        for (int nj = 0; nj < WN; ++nj)
            ob[st][nj] = BK ? ksz_off<true>(pc * N + col0 + 8 * nj + g, 2 * t + st, 0, 0)
                            : ksz_off<false>(col0 + 8 * nj + g, 2 * t + st, p.b_pitch, pc * kc);
    }
    const double ar = p.alpha, ai = p.alpha_i, br = p.beta, bi = p.beta_i;
    const int64_t scb = p.sC * 16;
    const uint32_t ring_off = (uint32_t)(ks_ring(smem) - smem);
    const bool tile_ok = pl < P;

    int s = 0;
    uint32_t phase = 0;
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int64_t b0 = u * P;
        const bool active = tile_ok && (b0 + pl) < batch;
        double re[WM][WN][2], im[WM][WN][2];
#pragma unroll
        for (int mi = 0; mi < WM; ++mi)
#pragma unroll
            for (int nj = 0; nj < WN; ++nj) re[mi][nj][0] = re[mi][nj][1] = im[mi][nj][0] = im[mi][nj][1] = 0.0;
        for (int ch = 0; ch < nchunks; ++ch) {
            mbar_wait(&full[s], phase);
            if (active) {
                const unsigned char *sa = smem + ring_off + (uint32_t)(s * stage_bytes);
                const unsigned char *sb = sa + a_bytes;
                const int kv = min(kc, K - ch * kc);
                const int nst = kv > 1 ? 2 : 1;  // step s covers k = 2t + s: all of kv when s < 2 and t < 4
#pragma unroll 2
                for (int st = 0; st < nst; ++st) {
                    double2 af[WM], bf[WN];
#pragma unroll
                    for (int mi = 0; mi < WM; ++mi) af[mi] = *reinterpret_cast<const double2 *>(sa + oa[st][mi]);
#pragma unroll
                    for (int nj = 0; nj < WN; ++nj) bf[nj] = *reinterpret_cast<const double2 *>(sb + ob[st][nj]);
#pragma unroll
                    for (int nj = 0; nj < WN; ++nj) {
                        const double nbi = -bf[nj].y;
#pragma unroll
                        for (int mi = 0; mi < WM; ++mi) {
                            ks_dmma_8x8x4(re[mi][nj][0], re[mi][nj][1], bf[nj].x, af[mi].x);
                            ks_dmma_8x8x4(re[mi][nj][0], re[mi][nj][1], nbi, af[mi].y);
                            ks_dmma_8x8x4(im[mi][nj][0], im[mi][nj][1], bf[nj].y, af[mi].x);
                            ks_dmma_8x8x4(im[mi][nj][0], im[mi][nj][1], bf[nj].x, af[mi].y);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == S) {
                s = 0;
                phase ^= 1u;
            }
        }
        if (active) {
            double *C = reinterpret_cast<double *>(p.C + (b0 + pl) * scb);
            // blocks in pairs: the pair's four C_in loads before its four stores
            // (stores may alias later loads, so each batch is one L2 round trip;
            // pairs halve the round trips at four more live doubles)
            // (single blocks for the largest tiles, whose accumulators leave no room)
            constexpr int NBLK = WM * WN, NB = NBLK <= 8 ? 2 : 1;
#pragma unroll
            for (int b0k = 0; b0k < NBLK; b0k += NB) {
                double2 ci[NB][2];
                double *q[NB];
#pragma unroll
                for (int u = 0; u < NB; ++u) {
                    const int bk = b0k + u < NBLK ? b0k + u : b0k;
                    const int mi = bk / WN, nj = bk % WN;
                    q[u] = C + 2 * ((row0 + 8 * mi + 2 * t) + (int64_t)(col0 + 8 * nj + g) * ldc);
                    if (!beta_zero && b0k + u < NBLK) {
                        ci[u][0] = __ldcs(reinterpret_cast<const double2 *>(q[u]));
                        ci[u][1] = __ldcs(reinterpret_cast<const double2 *>(q[u] + 2));
                    }
                }
#pragma unroll
                for (int u = 0; u < NB; ++u) {
                    if (b0k + u >= NBLK) break;
                    const int mi = (b0k + u) / WN, nj = (b0k + u) % WN;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const double sr = re[mi][nj][h], si = im[mi][nj][h];
                        double tr = 0.0, tim = 0.0;
                        if (!beta_zero) {
                            tr = fma_rn(br, ci[u][h].x, mul_rn(-bi, ci[u][h].y));
                            tim = fma_rn(br, ci[u][h].y, mul_rn(bi, ci[u][h].x));
                        }
                        double2 o;
                        o.x = fma_rn(ar, sr, fma_rn(-ai, si, tr));
                        o.y = fma_rn(ar, si, fma_rn(ai, sr, tim));
                        __stcs(reinterpret_cast<double2 *>(q[u] + 2 * h), o);
                    }
                }
            }
        }
    }
}

// ------------------------------------------------------------------ kernel body
// SINGLE: the plan has one tile class (single-class kernels) -- its fields
// are then read straight from the constant bank instead of through a
// dynamically indexed class table (registers).
template <typename T, bool TA, bool TB, typename Dispatcher, bool SINGLE = false>
__device__ __forceinline__ void ks_kernel_body(const CUtensorMap *tmA, const CUtensorMap *tmB,
                                               const IaatKsParams &p)
{
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + IAAT_KS_MAX_STAGES;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < p.S; ++s) {
            mbar_init(&full[s], p.ldgsts ? 32 : 1);
            mbar_init(&empty[s], p.n_compute_warps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    pdl_wait_and_release();
    if (warp == p.n_compute_warps) {
        if (p.ldgsts)
            ks_producer_ldgsts<T, TA, TB>(p, smem, full, empty, lane);
        else
            ks_producer<T, TA, TB>(p, tmA, tmB, smem, full, empty, lane);
        return;
    }
    if (SINGLE) {
        Dispatcher::run(p, p.cls[0], smem, full, empty, warp, lane);
        return;
    }
    int c = 0;
#pragma unroll
    for (int q = 1; q < IAAT_MAX_CLASSES; ++q)
        if (q < p.nclasses && warp >= p.cls[q].warp_begin) c = q;
    Dispatcher::run(p, p.cls[c], smem, full, empty, warp, lane);
}

}  // namespace iaat
