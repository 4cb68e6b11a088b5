// iaat_ksg.cuh -- the K-streamed "group" family (ksg): fp32 micro-kernels for
// the upper half of the small-GEMM domain (n >= ~40), B200 sm_100a.
//
// Why a third family.  On B200 a CUDA-core FFMA GEMM is bound by the bytes
// each lane pulls out of shared memory: the smem pipe delivers 128 B/clk
// per SM whether or not lanes share addresses (a warp-wide LDS.128 costs
// four wavefronts even as a broadcast), while the FMA pipes consume 128
// FMA/clk.  A lane with an mr x nr register tile loads (mr + nr) words per
// k-step for mr*nr FMAs, so at full FMA rate the smem pipe is
// 4(mr + nr)/(mr nr) busy: 1.0 for 8x8, 1.2 for 10x5, 0.8 for 10x10 -- the
// GPU form of the paper's "ratio of loads to FMAs", and
// the reason the round-1 slab/ks kernels (8x8 and smaller private tiles)
// stall at ~50 % of the FMA pipe for n >= 64.  ksg therefore runs the
// largest register tiles that fit (up to 128 accumulators), and:
//   * lane grids.  A warp owns one (LR*MR) x (LC*NR) block of ONE problem,
//     lanes laid out LR x LC (LR * LC = 32) over its tiles (the LC lanes of
//     a lane row share A fragments, the LR lanes of a lane column B
//     fragments: broadcasts, no bank conflicts).
//   * warp groups.  The consumer warps form G groups of W warps; each group
//     owns its own S-stage ring, its own producer warp, its own C buffer
//     and every G-th unit of P problems, so the groups drift apart and one
//     group's epilogue overlaps the other groups' FFMA2 main loops (the
//     ping-pang of PAPER.md:181 at the level of whole units).
//   * C through shared memory.  The producer TMA-loads C_in of a unit into
//     the group's C buffer while the unit's k loop runs, the epilogue
//     updates it in place (C = alpha*acc + beta*C_in) and the producer
//     TMA-stores the box: no lane waits on a global round trip, stores are
//     whole 128-byte lines, and the buffer's column pitch is padded (free:
//     the padding rows are out of the tensor, zero-filled on load and
//     clipped on store) so the epilogue's smem accesses are conflict-free.
//   * boundary by the copy engine.  The planner tiles an Mv x Nv problem
//     (Mv >= M, Nv >= N); the TMA boxes cover Mv / Nv, so rows and columns
//     past the problem arrive as zeros and are clipped from the C store --
//     no predicated code anywhere.  The planner weighs those idle FMAs
//     against the exact-tile families (it uses Mv = M, Nv = N whenever an
//     exact lane grid exists: "no boundary processing").
//
// Staging (no pack pass): one 3-D TMA box per operand per
// K-chunk of KC = 32 (128-byte swizzle) or 16 (64-byte swizzle) elements,
// straight from the caller's layout.  Element maps of a lane's tile inside
// its warp block (ti = lane % LR, tj = lane / LR):
//   K-major dim (rows of op(A) when transA = T, columns of op(B) when
//     transB = N):   element r at  t + L*r          (interleaved; consecutive
//                    lanes read consecutive swizzled rows: conflict-free)
//   MN-major dim:    element r at  V*(t + L*(r/V)) + r%V   (V-wide vector
//                    groups, neighbouring lanes read neighbouring vectors)
// Accumulation: one k-ascending FFMA (FFMA2 lane) chain per element, like
// every other fp32 kernel of the library -- results are bitwise identical
// across families and plans.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "iaat_device.cuh"
#include "iaat_params.h"

namespace iaat {
namespace ksg {

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2,
                                            uint32_t bar, uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap *map, uint32_t src, int c0, int c1, int c2)
{
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ float lds32(uint32_t a)
{
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void lds64(uint32_t a, float &x, float &y)
{
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(a));
}
__device__ __forceinline__ void lds128(uint32_t a, float &x, float &y, float &z, float &w)
{
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a));
}
__device__ __forceinline__ void sts32(uint32_t a, float x) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(x) : "memory"); }
__device__ __forceinline__ void sts64(uint32_t a, float x, float y)
{
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(x), "f"(y) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t a, float x, float y, float z, float w)
{
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}

// Lane-grid geometry of one class.  PV (column-pair boxes, IaatKsgParams::
// pairv): column pitches are 8-byte, not 16-byte, multiples, so MN-major
// vector groups are at most 2 wide.
template <bool TA, bool TB, int MR, int NR, int LR, bool PV = false>
struct Geo {
    static constexpr int LC = 32 / LR;
    static constexpr bool AK = TA;   // op(A) K-major in smem
    static constexpr bool BK = !TB;  // op(B) K-major in smem
    static constexpr int VA = AK ? 1 : ((MR % 4 == 0 && !PV) ? 4 : (MR % 2 == 0 ? 2 : 1));
    static constexpr int VB = BK ? 1 : ((NR % 4 == 0 && !PV) ? 4 : (NR % 2 == 0 ? 2 : 1));
    // FFMA2 pairs along the dim whose fragments arrive as vectors
    static constexpr int PAIR = (!AK && VA >= 2) ? 1 : ((!BK && VB >= 2) ? 2 : 0);
    static constexpr int BR = LR * MR;  // warp block rows
    static constexpr int BC = LC * NR;  // warp block columns
    // PV column map: the C buffer's columns are M = 2 (mod 4) words apart and
    // cannot be padded, so neighbouring lanes must sit FOUR columns apart
    // (4 M = 8 or 24 mod 32: a quarter-warp's 8-word row groups fall in
    // disjoint banks; one column apart they overlap 2-4 ways).  A lane owns
    // groups of 4 adjacent columns, 4 LC apart; the NR % 4 left-over columns
    // sit after the groups, NR % 4 per lane.
    static constexpr int NG = NR / 4 * 4, RB = NR % 4;
    __device__ static __forceinline__ int row(int ti, int r) { return AK ? ti + LR * r : VA * (ti + LR * (r / VA)) + r % VA; }
    __device__ static __forceinline__ int col(int tj, int c)
    {
        if (PV) return c < NG ? 4 * LC * (c / 4) + 4 * tj + c % 4 : LC * NG + RB * tj + (c - NG);
        return BK ? tj + LC * c : VB * (tj + LC * (c / VB)) + c % VB;
    }
};

// Swizzled K-major row base: 16-byte chunk q of smem row ra (KC*4 bytes,
// 128- or 64-byte TMA swizzle) lives at (kmaj_base(ra) ^ (q << 4)).
template <int KC>
__device__ __forceinline__ uint32_t kmaj_base(int ra)
{
    if (KC == 32) return ((uint32_t)ra << 7) | ((uint32_t)(ra & 7) << 4);
    return ((uint32_t)ra << 6) | ((uint32_t)((ra >> 1) & 3) << 4);
}

// Fragment of one operand for one k-block of KU (1, 2 or 4) k-steps: f[kk][r].
// K-major: one LDS.32 / LDS.64 / LDS.128 per element row (KU consecutive k values);
// MN-major: one V-wide load per vector group per k-step.
// K-major rows of a lane are L apart; when L is a multiple of 8 every row
// of the lane has the same swizzle phase (the 128-byte swizzle repeats every
// 8 rows, the 64-byte one every 8 rows of 64 bytes), so one XOR on the first
// row's base serves all rows and the rest are immediates (UNI): no per-row
// LOP3 / IADD in the k loop (measured: the general path made NN / TT loops
// ~9 % slower than NT's, which has no K-major operand).
// PV (column-pair boxes), K-major: the even and the odd columns of the
// operand arrive as two unswizzled half boxes with rows of KC + 4 elements
// (TMA box starts must be 16-byte aligned -- measured: an 8-byte-aligned
// inner coordinate faults -- so the odd columns' box starts ld % 4 elements
// early and their k values sit that far into the row).  A lane's rows all
// have the parity of its first row: they sit L / 2 rows apart in one half
// box, at immediates from base[0]; the 8-byte row offsets allow LDS.64, and
// rows 20 / 36 words apart keep a quarter-warp's pairs in distinct banks.
template <bool KMAJ, int R, int V, int L, int KC, bool PV = false>
struct Opnd {
    static constexpr bool UNI = KMAJ && (L % 8 == 0) && !PV;
    static constexpr uint32_t PSTEP = (uint32_t)((L / 2) * (KC + 4) * 4);  // PV K-major: bytes between a lane's rows
    uint32_t base[KMAJ ? R : 1];  // K-major: per-row swizzled base; MN-major: first element
    uint32_t pitch;               // MN-major: bytes per k-step
    template <int KU>
    __device__ __forceinline__ void load(float (&f)[KU][R], uint32_t stage, int kb) const
    {
        if (PV && KMAJ) {
            const uint32_t x = stage + base[0] + (uint32_t)kb * 4u;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t a = x + (uint32_t)r * PSTEP;
                if (KU == 4) {
                    lds64(a, f[0][r], f[KU > 1 ? 1 : 0][r]);
                    lds64(a + 8, f[KU > 2 ? 2 : 0][r], f[KU > 3 ? 3 : 0][r]);
                } else if (KU == 2) {
                    lds64(a, f[0][r], f[KU > 1 ? 1 : 0][r]);
                } else {
                    f[0][r] = lds32(a);
                }
            }
        } else if (UNI) {
            const uint32_t q = (uint32_t)(kb >> 2) << 4, w = (uint32_t)(kb & 3) * 4u;
            const uint32_t x = stage + (base[0] ^ q) + (KU == 4 ? 0u : w);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t a = x + (uint32_t)(r * L * KC * 4);
                if (KU == 4) lds128(a, f[0][r], f[KU > 1 ? 1 : 0][r], f[KU > 2 ? 2 : 0][r], f[KU > 3 ? 3 : 0][r]);
                else if (KU == 2) lds64(a, f[0][r], f[KU > 1 ? 1 : 0][r]);
                else f[0][r] = lds32(a);
            }
        } else if (KMAJ) {
            const uint32_t q = (uint32_t)(kb >> 2) << 4, w = (uint32_t)(kb & 3) * 4u;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (KU == 4) lds128(stage + (base[r] ^ q), f[0][r], f[KU > 1 ? 1 : 0][r], f[KU > 2 ? 2 : 0][r], f[KU > 3 ? 3 : 0][r]);
                else if (KU == 2) lds64(stage + (base[r] ^ q) + w, f[0][r], f[KU > 1 ? 1 : 0][r]);
                else f[0][r] = lds32(stage + (base[r] ^ q) + w);
            }
        } else {
#pragma unroll
            for (int kk = 0; kk < KU; ++kk) {
                const uint32_t a = stage + base[0] + (uint32_t)(kb + kk) * pitch;
#pragma unroll
                for (int g = 0; g < R / V; ++g) {
                    const uint32_t ag = a + (uint32_t)(g * V * L * 4);
                    if (V == 4) lds128(ag, f[kk][4 * g], f[kk][4 * g + 1], f[kk][4 * g + 2], f[kk][4 * g + 3]);
                    else if (V == 2) lds64(ag, f[kk][2 * g], f[kk][2 * g + 1]);
                    else f[kk][g] = lds32(ag);
                }
            }
        }
    }
    // one k-step (ragged chunk tails)
    __device__ __forceinline__ void load1(float (&f)[R], uint32_t stage, int k) const
    {
        if (PV && KMAJ) {
#pragma unroll
            for (int r = 0; r < R; ++r) f[r] = lds32(stage + base[0] + (uint32_t)k * 4u + (uint32_t)r * PSTEP);
        } else if (KMAJ) {
            const uint32_t q = (uint32_t)(k >> 2) << 4, w = (uint32_t)(k & 3) * 4u;
#pragma unroll
            for (int r = 0; r < R; ++r) f[r] = lds32(stage + (base[r] ^ q) + w);
        } else {
            const uint32_t a = stage + base[0] + (uint32_t)k * pitch;
#pragma unroll
            for (int r = 0; r < R; ++r) f[r] = lds32(a + (uint32_t)(((r / V) * V * L + r % V) * 4));
        }
    }
};

// PV: op(B)'s fragment loads under Geo's PV column map (col = 4 LC g + 4 tj + j
// for the grouped columns, LC NG + RB tj + j' for the NR % 4 left-over ones).
// K-major (two unswizzled half boxes, rows of KC + 4 elements): a grouped
// column's parity is j's, so two bases (even / odd half) + immediates serve
// them; the left-over columns keep one byte offset each.  MN-major (pitch ld,
// 8-byte aligned columns): one base for the groups, one for the left-overs.
template <bool KMAJ, int R, int V, int L, int KC>
struct OpndPV {
    static constexpr int NG = R / 4 * 4, RB = R % 4;
    static constexpr uint32_t RP = (uint32_t)((KC + 4) * 4);  // K-major: bytes per smem row
    uint32_t be[2];                 // K-major: even / odd half base of the lane's groups; MN-major: be[0] = groups, be[1] = left-overs
    uint32_t brem[RB ? RB : 1];     // K-major: byte offset of each left-over column
    uint32_t pitch;                 // MN-major: bytes per k-step
    // x0: first column of the warp block (C0), t: the lane's tj, pl: problem, ext: Nv
    __device__ __forceinline__ void setup(int x0, int t, int pl, int ext, int half, int ld, int kcpitch)
    {
        if (KMAJ) {
            be[0] = (uint32_t)(pl * (ext >> 1) + (x0 >> 1) + 2 * t) * RP;
            be[1] = be[0] + (uint32_t)(half + (ld & 3) * 4);
#pragma unroll
            for (int j = 0; j < RB; ++j) {
                const int x = x0 + L * NG + RB * t + j;
                brem[j] = (uint32_t)((x & 1) * (half + (ld & 3) * 4)) + (uint32_t)(pl * (ext >> 1) + (x >> 1)) * RP;
            }
        } else {
            be[0] = (uint32_t)((pl * kcpitch + x0 + 4 * t) * 4);
            be[1] = (uint32_t)((pl * kcpitch + x0 + L * NG + RB * t) * 4);
        }
    }
    // byte address of column c at k-step 0 of the stage (K-major) / element c of k-step row a (MN-major)
    __device__ __forceinline__ uint32_t kaddr(uint32_t stage, int c) const
    {
        return c < NG ? stage + be[c & 1] + (uint32_t)(2 * L * (c / 4) + ((c % 4) >> 1)) * RP : stage + brem[c < NG ? 0 : c - NG];
    }
    __device__ __forceinline__ uint32_t maddr(uint32_t a, int c) const
    {
        return c < NG ? a + be[0] + (uint32_t)((4 * L * (c / 4) + c % 4) * 4) : a + be[1] + (uint32_t)((c - NG) * 4);
    }
    template <int KU>
    __device__ __forceinline__ void load(float (&f)[KU][R], uint32_t stage, int kb) const
    {
        if (KMAJ) {
#pragma unroll
            for (int c = 0; c < R; ++c) {
                const uint32_t a = kaddr(stage, c) + (uint32_t)kb * 4u;
                if (KU == 4) {
                    lds64(a, f[0][c], f[KU > 1 ? 1 : 0][c]);
                    lds64(a + 8, f[KU > 2 ? 2 : 0][c], f[KU > 3 ? 3 : 0][c]);
                } else if (KU == 2) {
                    lds64(a, f[0][c], f[KU > 1 ? 1 : 0][c]);
                } else {
                    f[0][c] = lds32(a);
                }
            }
        } else {
#pragma unroll
            for (int kk = 0; kk < KU; ++kk) {
                const uint32_t a = stage + (uint32_t)(kb + kk) * pitch;
#pragma unroll
                for (int c = 0; c < R; c += V) {
                    if (V == 2) lds64(maddr(a, c), f[kk][c], f[kk][c + 1 < R ? c + 1 : c]);
                    else f[kk][c] = lds32(maddr(a, c));
                }
            }
        }
    }
    __device__ __forceinline__ void load1(float (&f)[R], uint32_t stage, int k) const
    {
#pragma unroll
        for (int c = 0; c < R; ++c)
            f[c] = KMAJ ? lds32(kaddr(stage, c) + (uint32_t)k * 4u) : lds32(maddr(stage + (uint32_t)k * pitch, c));
    }
};

template <bool PV, typename A, typename B>
struct SelOpnd {
    typedef B type;
};
template <typename A, typename B>
struct SelOpnd<true, A, B> {
    typedef A type;
};

#ifndef IAAT_KSG_EVICT_FIRST
#define IAAT_KSG_EVICT_FIRST 0
#endif
#ifndef IAAT_KSG_FMA_ORDER
#define IAAT_KSG_FMA_ORDER 1
#endif
template <int KU, int MR, int NR, int PAIR>
__device__ __forceinline__ void kblock_fma(RegTile<float, MR, NR, PAIR> &acc, const float (&a)[KU][MR],
                                           const float (&b)[KU][NR])
{
    if constexpr (PAIR == 1 && IAAT_KSG_FMA_ORDER == 1) {
        // pair-outer order: consecutive FFMA2s share the a-pair operand
#pragma unroll
        for (int kk = 0; kk < KU; ++kk)
#pragma unroll
            for (int i = 0; i < MR / 2; ++i) {
                const unsigned long long ap = pack_f32x2(a[kk][2 * i], a[kk][2 * i + 1]);
#pragma unroll
                for (int j = 0; j < NR; ++j) ffma2(acc.v[i][j], ap, pack_f32x2(b[kk][j], b[kk][j]));
            }
    } else {
#pragma unroll
        for (int kk = 0; kk < KU; ++kk) acc.rank1([&](int i) { return a[kk][i]; }, [&](int j) { return b[kk][j]; });
    }
}

// Shared-memory map: [barriers (1 KB)] then, per group g, at the first
// 1024-byte boundary after them + g * group_bytes: S stages of
// [A box | B box], then the C buffer (one TMA box [P][Nv][c_pitch] of C).
struct Smem {
    uint32_t ring;  // shared address of the group's stage 0
    uint32_t cbuf;  // shared address of the group's C buffer
    uint32_t full, empty, cfull, cready;  // shared addresses of the group's mbarriers
    __device__ __forceinline__ Smem(unsigned char *smem, const IaatKsgParams &p, int g)
    {
        const uint32_t sbase = smem_u32(smem);
        ring = ((sbase + IAAT_KSG_BAR_BYTES + 1023u) & ~1023u) + (uint32_t)g * (uint32_t)p.group_bytes;
        cbuf = ring + (uint32_t)(p.S * p.stage_bytes);
        full = sbase + (uint32_t)(g * IAAT_KSG_GROUP_BARS * 8);
        empty = full + IAAT_KSG_MAX_STAGES * 8;
        cfull = empty + IAAT_KSG_MAX_STAGES * 8;
        cready = cfull + 8;
    }
};

__device__ __forceinline__ void bar_init(uint32_t b, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint32_t b)
{
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint32_t b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t b, uint32_t parity)
{
    uint32_t ok;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(b), "r"(parity)
            : "memory");
    } while (!ok);
}

// Consumer warp: one warp block of one problem per unit of its group.
// DBG (experiment builds only; the library instantiates DBG = 0):
//   bit 0: no A/B staging (consumers never wait for or release stages),
//   bit 1: no epilogue (no C load / update / store).
template <bool TA, bool TB, int MR, int NR, int LR, int KC, int KU, int G, int W, int DBG = 0, bool PV = false>
__device__ __forceinline__ void ksg_consumer(const IaatKsgParams &p, unsigned char *smem, int g, int w, int lane)
{
    typedef Geo<TA, TB, MR, NR, LR, PV> Gm;
    constexpr bool AK = Gm::AK, BK = Gm::BK;
    const int K = p.K, nchunks = p.nchunks, S = p.S, Mv = p.Mv, Nv = p.Nv, cp = p.c_pitch;
    const int64_t nunits = p.nunits;
    const int ti = lane % LR, tj = lane / LR;
    const int pl = w / p.wpp, blk = w - pl * p.wpp;
    const int R0 = (blk % p.bm) * Gm::BR, C0 = (blk / p.bm) * Gm::BC;
    const Smem sm(smem, p, g);

    Opnd<AK, MR, Gm::VA, LR, KC, PV> oa;
    typename SelOpnd<PV, OpndPV<BK, NR, Gm::VB, Gm::LC, KC>, Opnd<BK, NR, Gm::VB, Gm::LC, KC, false>>::type ob;
    // PV: byte offset of K-major row / column x of problem pl -- even ones in
    // the first half box, odd ones in the second, ld % 4 elements into the row
    auto pvrow = [&](int x, int ext, int half, int ld) {
        return (uint32_t)((x & 1) * (half + (ld & 3) * 4) + (pl * (ext >> 1) + (x >> 1)) * (KC + 4) * 4);
    };
    if (AK && PV) {
        oa.base[0] = pvrow(R0 + Gm::row(ti, 0), Mv, p.a_half, p.lda);
    } else if (AK) {
#pragma unroll
        for (int r = 0; r < MR; ++r) oa.base[r] = kmaj_base<KC>(pl * Mv + R0 + Gm::row(ti, r));
    } else {
        oa.base[0] = (uint32_t)((pl * KC * p.a_pitch + R0 + Gm::VA * ti) * 4);
    }
    if constexpr (PV) {
        ob.setup(C0, tj, pl, Nv, p.b_half, p.ldb, KC * p.b_pitch);
    } else if constexpr (BK) {
#pragma unroll
        for (int c = 0; c < NR; ++c) ob.base[c] = kmaj_base<KC>(pl * Nv + C0 + Gm::col(tj, c));
    } else {
        ob.base[0] = (uint32_t)((pl * KC * p.b_pitch + C0 + Gm::VB * tj) * 4);
    }
    oa.pitch = (uint32_t)p.a_pitch * 4u;
    ob.pitch = (uint32_t)p.b_pitch * 4u;
    const float alpha = (float)p.alpha, beta = (float)p.beta;
    const bool beta_zero = p.beta_zero != 0;
    // this warp block's first C element in the group's C buffer
    const uint32_t cb0 = sm.cbuf + (uint32_t)(((pl * Nv + C0) * cp + R0) * 4);
    // PV: the C buffer's columns are M apart, so a row past M would land in
    // the next column: the only boundary code, one predicate per store
    const int mrows = PV ? p.M - R0 : (1 << 30);

    int s = 0;
    uint32_t phase = 0, cphase = 0;
    for (int64_t u = (int64_t)blockIdx.x * G + g; u < nunits; u += (int64_t)gridDim.x * G) {
        RegTile<float, MR, NR, Gm::PAIR> acc;
        acc.zero();
        for (int ch = 0; ch < nchunks; ++ch) {
            if (!(DBG & 1)) bar_wait(sm.full + 8 * s, phase);
            const uint32_t sa = sm.ring + (uint32_t)(s * p.stage_bytes), sb = sa + (uint32_t)p.a_bytes;
            const int kv = min(KC, K - ch * KC);
            if (kv == KC) {
                // register double buffering (the paper's ping-pang,
                // PAPER.md:181): the fragments of k-block kb + KU load while
                // the FFMA2s of kb issue
                float fa[2][KU][MR], fb[2][KU][NR];
                oa.template load<KU>(fa[0], sa, 0);
                ob.template load<KU>(fb[0], sb, 0);
#pragma unroll
                for (int kb = 0; kb < KC; kb += KU) {
                    const int cur = (kb / KU) & 1;
                    if (kb + KU < KC) {
                        oa.template load<KU>(fa[cur ^ 1], sa, kb + KU);
                        ob.template load<KU>(fb[cur ^ 1], sb, kb + KU);
                    }
                    kblock_fma<KU, MR, NR, Gm::PAIR>(acc, fa[cur], fb[cur]);
                }
            } else {
                // (ragged last chunk: software-pipelined pieces of 16 / 8 / 4
                // k-steps instead of this loop measured neutral -- n = 76
                // entry 0 95.2 us either way, r2s4_g7 -- the chunk is FMA-bound)
                int kb = 0;
#pragma unroll 1
                for (; kb + 4 <= kv; kb += 4) {
                    float fa[4][MR], fb[4][NR];
                    oa.template load<4>(fa, sa, kb);
                    ob.template load<4>(fb, sb, kb);
                    kblock_fma<4, MR, NR, Gm::PAIR>(acc, fa, fb);
                }
#pragma unroll 1
                for (; kb < kv; ++kb) {
                    float a1[MR], b1[NR];
                    oa.load1(a1, sa, kb);
                    ob.load1(b1, sb, kb);
                    acc.rank1([&](int i) { return a1[i]; }, [&](int j) { return b1[j]; });
                }
            }
            __syncwarp();
            if (lane == 0 && !(DBG & 1)) bar_arrive(sm.empty + 8 * s);
            if (++s == S) {
                s = 0;
                phase ^= 1u;
            }
        }
        // fused epilogue in the group's C buffer (C_in already there when
        // beta != 0): C = fma(alpha, acc, beta*C_in) -- the same two
        // roundings as every other family's epilogue, so results stay
        // bitwise identical across plans -- written back in place; the
        // producer then TMA-stores the box.
        if (DBG & 2) {
            float v[MR][NR];
            acc.get(v);
            float t = 0.f;
#pragma unroll
            for (int c = 0; c < NR; ++c)
#pragma unroll
                for (int r = 0; r < MR; ++r) t += v[r][c];
            if (t == 1234.5f) sts32(sm.cbuf, t);
            continue;
        }
        bar_wait(sm.cfull, cphase);
        cphase ^= 1u;
        if constexpr (Gm::PAIR == 1 && !AK && Gm::VA == 2) {
            // accumulator pairs are two adjacent C rows: one LDS.64 of C_in,
            // FMUL2 + FFMA2 (the same two IEEE roundings per element), one STS.64
            const unsigned long long a2 = pack_f32x2(alpha, alpha), b2 = pack_f32x2(beta, beta);
#pragma unroll
            for (int c = 0; c < NR; ++c) {
                const uint32_t colb = cb0 + (uint32_t)(Gm::col(tj, c) * cp * 4);
#pragma unroll
                for (int q = 0; q < MR / 2; ++q) {
                    const uint32_t a = colb + (uint32_t)(Gm::row(ti, 2 * q) * 4);
                    if (PV && Gm::row(ti, 2 * q) >= mrows) continue;
                    unsigned long long o;
                    if (beta_zero) {
                        asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(o) : "l"(a2), "l"(acc.v[q][c]));
                    } else {
                        unsigned long long ci, t;
                        asm volatile("ld.shared.b64 %0, [%1];" : "=l"(ci) : "r"(a));
                        asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(b2), "l"(ci));
                        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(o) : "l"(a2), "l"(acc.v[q][c]), "l"(t));
                    }
                    asm volatile("st.shared.b64 [%0], %1;" ::"r"(a), "l"(o) : "memory");
                }
            }
        } else {
            float v[MR][NR];
            acc.get(v);
#pragma unroll
            for (int c = 0; c < NR; ++c) {
                const uint32_t colb = cb0 + (uint32_t)(Gm::col(tj, c) * cp * 4);
                if (!AK && Gm::VA >= 2) {
#pragma unroll
                    for (int g4 = 0; g4 < MR / Gm::VA; ++g4) {
                        const uint32_t q = colb + (uint32_t)(Gm::row(ti, Gm::VA * g4) * 4);
                        if (PV && Gm::row(ti, Gm::VA * g4) >= mrows) continue;
                        float ci[4] = {0.f, 0.f, 0.f, 0.f}, o[4];
                        if (!beta_zero) {
                            if (Gm::VA == 4) lds128(q, ci[0], ci[1], ci[2], ci[3]);
                            else lds64(q, ci[0], ci[1]);
                        }
#pragma unroll
                        for (int e = 0; e < Gm::VA; ++e) {
                            const float x = v[Gm::VA * g4 + e][c];
                            o[e] = beta_zero ? mul_rn(alpha, x) : fma_rn(alpha, x, mul_rn(beta, ci[e]));
                        }
                        if (Gm::VA == 4) sts128(q, o[0], o[1], o[2], o[3]);
                        else sts64(q, o[0], o[1]);
                    }
                } else {
#pragma unroll
                    for (int r = 0; r < MR; ++r) {
                        const uint32_t q = colb + (uint32_t)(Gm::row(ti, r) * 4);
                        if (PV && Gm::row(ti, r) >= mrows) continue;
                        const float x = v[r][c];
                        sts32(q, beta_zero ? mul_rn(alpha, x) : fma_rn(alpha, x, mul_rn(beta, lds32(q))));
                    }
                }
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) bar_arrive(sm.cready);
    }
}

// Producer warp of group g: lane 0 streams the group's units chunk by chunk,
// and after each unit's chunks are queued it retires the previous unit's C
// (TMA store once its epilogue is done) and brings in this unit's C_in.
template <bool TA, bool TB, int KC, int G, int DBG = 0, bool PV = false>
__device__ __forceinline__ void ksg_producer(const IaatKsgParams &p, const CUtensorMap *tmA, const CUtensorMap *tmB,
                                             const CUtensorMap *tmC, unsigned char *smem, int g, int lane)
{
    if (lane != 0) return;
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmB)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmC)) : "memory");
    // L2 policies.  evict_first is right for data read once -- but a K-major
    // box row (kc * 4 = 64 or 128 bytes of one column) starts at the
    // column's own alignment, so consecutive K-chunks of a column share a
    // 32-byte sector at their boundary; with evict_first that sector is gone
    // before the next chunk's load and is read twice (ncu: DRAM reads +9-17 %
    // over the operand bytes at n = 56-76).  K-major operands therefore load
    // with normal priority (measured +5 % at n = 56 NN / TT); MN-major boxes
    // (whole contiguous rows) and C keep evict_first.
    const uint64_t pol = policy_evict_first();
    uint64_t pol_norm;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_norm));
    const uint64_t polA = (TA && !IAAT_KSG_EVICT_FIRST) ? pol_norm : pol;
    const uint64_t polB = (!TB && !IAAT_KSG_EVICT_FIRST) ? pol_norm : pol;
    const uint32_t tx = (uint32_t)(p.a_tx + p.b_tx);
    const Smem sm(smem, p, g);
    int s = 0, it = 0;
    uint32_t phase = 0, rphase = 0;
    int prev_b0 = -1;
    auto issue_chunk = [&](int b0, int c) {
        if (it >= p.S) bar_wait(sm.empty + 8 * s, phase);
        const uint32_t st = sm.ring + (uint32_t)(s * p.stage_bytes), fb = sm.full + 8 * s;
        bar_expect_tx(fb, tx);
        const int k0 = c * KC;
        if (PV) {
            // column-pair boxes: an MN-major operand's K-chunk is KC / 2 pair
            // rows; a K-major one's is two boxes of KC + 4 elements, the even
            // columns (the first ld elements of the pair rows) and the odd
            // ones (the next ld; box start rounded down to 16 bytes)
            if (TA) {
                tma_load_3d(st, tmA, k0, 0, b0, fb, polA);
                tma_load_3d(st + (uint32_t)p.a_half, tmA, p.lda + k0 - (p.lda & 3), 0, b0, fb, polA);
            } else {
                tma_load_3d(st, tmA, 0, k0 >> 1, b0, fb, polA);
            }
            if (TB) {
                tma_load_3d(st + p.a_bytes, tmB, 0, k0 >> 1, b0, fb, polB);
            } else {
                tma_load_3d(st + p.a_bytes, tmB, k0, 0, b0, fb, polB);
                tma_load_3d(st + p.a_bytes + (uint32_t)p.b_half, tmB, p.ldb + k0 - (p.ldb & 3), 0, b0, fb, polB);
            }
        } else {
            if (TA) tma_load_3d(st, tmA, k0, 0, b0, fb, polA);
            else tma_load_3d(st, tmA, 0, k0, b0, fb, polA);
            if (TB) tma_load_3d(st + p.a_bytes, tmB, 0, k0, b0, fb, polB);
            else tma_load_3d(st + p.a_bytes, tmB, k0, 0, b0, fb, polB);
        }
        if (++s == p.S) {
            s = 0;
            if (it >= 2 * p.S - 1) phase ^= 1u;
        }
        ++it;
    };
    const int nch = (DBG & 1) ? 0 : p.nchunks;
    for (int64_t u = (int64_t)blockIdx.x * G + g; u < p.nunits; u += (int64_t)gridDim.x * G) {
        const int b0 = (int)(u * p.P);
        // the first ring's worth of this unit's chunks (their slots free up
        // as the previous unit's k loop ends), then the previous unit's C
        // (stored as soon as its epilogue is done) and this unit's C_in --
        // early, so that both overlap this unit's k loop -- then the rest
        int c = 0;
        for (; c < min(p.S, nch); ++c) issue_chunk(b0, c);
        if (!(DBG & 2)) {
            if (prev_b0 >= 0) {
                bar_wait(sm.cready, rphase);
                rphase ^= 1u;
                tma_store_3d(tmC, sm.cbuf, 0, 0, prev_b0);
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            if (!p.beta_zero) {
                bar_expect_tx(sm.cfull, (uint32_t)p.c_tx);
                tma_load_3d(sm.cbuf, tmC, 0, 0, b0, sm.cfull, pol);
            } else {
                bar_arrive(sm.cfull);
            }
            prev_b0 = b0;
        }
        for (; c < nch; ++c) issue_chunk(b0, c);
    }
    if (prev_b0 >= 0 && !(DBG & 2)) {
        bar_wait(sm.cready, rphase);
        tma_store_3d(tmC, sm.cbuf, 0, 0, prev_b0);
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

// The kernel body: 1 + G*W/4 warpgroups.  Warpgroup 0 holds the producers
// (warp g < G serves group g; the others retire at once) and gives
// registers back (setmaxnreg.dec); the G*W = 8 or 12 consumer warps take
// them (setmaxnreg.inc) for the register tiles.  Consumer c = warp - 4 is
// warp c % W of group c / W, so every SMSP (warp % 4) hosts warps of
// different groups.
#define IAAT_KSG_THREADS_OF(GW) (128 + 32 * (GW))
#define IAAT_KSG_PRODUCER_REGS 40
#define IAAT_KSG_CONSUMER_REGS_OF(GW) ((GW) == 8 ? 232 : 152)
template <bool TA, bool TB, int MR, int NR, int LR, int KC, int KU, int G, int W, int DBG = 0, bool PV = false>
__device__ __forceinline__ void ksg_body(const IaatKsgParams &p, const CUtensorMap *tmA, const CUtensorMap *tmB,
                                         const CUtensorMap *tmC)
{
    static_assert(G * W == 8 || G * W == 12, "ksg: two or three warpgroups of consumers");
    static_assert(G <= IAAT_KSG_MAX_GROUPS, "ksg: barrier area holds IAAT_KSG_MAX_GROUPS groups");
    extern __shared__ __align__(1024) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x < G) {
        const Smem sm(smem, p, threadIdx.x);
        for (int s = 0; s < p.S; ++s) {
            bar_init(sm.full + 8 * s, 1);
            bar_init(sm.empty + 8 * s, W);
        }
        bar_init(sm.cfull, 1);
        bar_init(sm.cready, W);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(IAAT_KSG_PRODUCER_REGS));
        if (warp < G) ksg_producer<TA, TB, KC, G, DBG, PV>(p, tmA, tmB, tmC, smem, warp, lane);
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(IAAT_KSG_CONSUMER_REGS_OF(G * W)));
        const int c = warp - 4;
        ksg_consumer<TA, TB, MR, NR, LR, KC, KU, G, W, DBG, PV>(p, smem, c / W, c % W, lane);
    }
}

}  // namespace ksg
}  // namespace iaat

// ======================================================================
// ksgs: the ksg lane grids on SLAB staging, for inputs the TMA rules
// exclude (odd ld's: config 3, M or N = 2 mod 4, misaligned bases).  A unit
// of P consecutive packed problems is one stage: ONE cp.async.bulk per
// operand of the 16-byte-aligned span enclosing the P problems' bytes (the
// slab family's staging, no pack pass), read in place with
// scalar LDS at any element alignment.  Tiles cover an Mv x Nv >= M x N
// block grid; rows / columns past M / N compute on whatever lies in the
// stage (the next column, the next problem or the slack) and are never
// stored: the only boundary code is the store predicate of the epilogue,
// once per element per unit.  C_in is read from global (L2-prefetched by
// the producer when the unit is staged), all of a lane's C_in loads issued
// before its first store.
// ======================================================================
namespace iaat {
namespace ksg {

template <bool TA, bool TB, int MR, int NR, int LR>
struct GeoS {
    static constexpr int LC = 32 / LR;
    static constexpr bool AK = TA, BK = !TB;
    // FFMA2 pairs: scalar loads put any two values in a register pair, so
    // either operand can supply the pairs -- the MN-major one when it can
    // (3 / 4: odd MR / NR, pairs for all but the last row / column)
    static constexpr int PAIR = (!AK && MR % 2 == 0) ? 1
                              : (!BK && NR % 2 == 0) ? 2
                              : (MR % 2 == 0) ? 1
                              : (NR % 2 == 0) ? 2
                              : (MR >= 3 && !AK) ? 3
                              : (NR >= 3) ? 4
                              : (MR >= 3) ? 3 : 0;
    static constexpr int BR = LR * MR, BC = LC * NR;
    __device__ static __forceinline__ int row(int ti, int r) { return ti + LR * r; }
    __device__ static __forceinline__ int col(int tj, int c) { return tj + LC * c; }
};

// Shared-memory map of ksgs: [full[S] | empty[S] barriers (1 KB)], then the
// ring of S stages [A span | B span] shared by all groups.
// ticket[s] = the unit sequence number j whose fill of stage s the producer
// has started (written after it saw the stage's previous fill consumed).
// Consecutive fills of a stage can belong to different groups, and an
// mbarrier parity wait cannot tell fill n from fill n - 2: a group that
// reached its wait for fill n while fill n - 1 was still pending would pass
// at once.  A consumer therefore first waits for ticket[s] == j; from then
// on the stage's barrier is in the phase of fill j / S.
struct SmemS {
    uint32_t ring, full, empty, ticket;
    __device__ __forceinline__ explicit SmemS(unsigned char *smem)
    {
        const uint32_t sbase = smem_u32(smem);
        ring = (sbase + IAAT_KSG_BAR_BYTES + 1023u) & ~1023u;
        full = sbase;
        empty = sbase + IAAT_KSGS_MAX_STAGES * 8;
        ticket = sbase + IAAT_KSGS_MAX_STAGES * 16;
    }
};

__device__ __forceinline__ void ticket_set(uint32_t a, int v)
{
    asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void ticket_wait(uint32_t a, int v)
{
    int t;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(t) : "r"(a) : "memory");
    while (t != v) {  // rare: the stage still holds an earlier unit; back off, leave the SMSP to the others
        __nanosleep(64);
        asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(t) : "r"(a) : "memory");
    }
}

template <bool TA, bool TB, int MR, int NR, int LR, int G, int W, bool CS>
__device__ __forceinline__ void ksgs_consumer(const IaatKsgParams &p, unsigned char *smem, int g, int w, int lane)
{
    typedef GeoS<TA, TB, MR, NR, LR> Gm;
    constexpr bool AK = Gm::AK, BK = Gm::BK;
    const int K = p.K, S = p.S, M = p.M, N = p.N, lda = p.lda, ldb = p.ldb, ldc = p.ldc;
    const int64_t nunits = p.nunits, batch = p.batch;
    const int ti = lane % LR, tj = lane / LR;
    const int pl = w / p.wpp, blk = w - pl * p.wpp;
    const int R0 = (blk % p.bm) * Gm::BR, C0 = (blk / p.bm) * Gm::BC;
    const SmemS sm(smem);
    const float alpha = (float)p.alpha, beta = (float)p.beta;
    const bool beta_zero = p.beta_zero != 0;
    // element offsets (words) of the lane's rows / columns inside its problem
    // (the k-independent part): MN-major rows / columns are contiguous words,
    // K-major ones are ld apart
    // ra / rb: byte address of each K-major row / column (of the first element
    // of an MN-major operand) at k = 0 of the current unit -- the element
    // offset here, the unit's stage address added before and taken off after
    // the unit's k loop.  One register per K-major row: inside
    // the unrolled k loop a load is [row + k * 4 + immediate], one add per
    // row per four k-steps.  (The earlier form, (k-dependent base) + 4 *
    // offset[r], cost one IMAD per row per k-step on the pipe the FFMA2s
    // need: 10 of 41 instructions per k-step of the TN 8x4 tile.)
    uint32_t ra[AK ? MR : 1], rb[BK ? NR : 1];
    if (AK) {
#pragma unroll
        for (int r = 0; r < MR; ++r) ra[r] = (uint32_t)((R0 + Gm::row(ti, r)) * lda * 4);
    } else {
        ra[0] = (uint32_t)((R0 + ti) * 4);
    }
    if (BK) {
#pragma unroll
        for (int c = 0; c < NR; ++c) rb[c] = (uint32_t)((C0 + Gm::col(tj, c)) * ldb * 4);
    } else {
        rb[0] = (uint32_t)((C0 + tj) * 4);
    }
    const int64_t sA = p.sA, sB = p.sB, sC = p.sC;

    // one ring of S stages shared by the G groups: the CTA's j-th unit
    // (j = 0, 1, ...; group j % G) sits in stage j % S, fill j / S
    int j = g;
    for (int64_t u = (int64_t)blockIdx.x * G + g; u < nunits; u += (int64_t)gridDim.x * G, j += G) {
        const int s = j % S;
        const uint32_t phase = (uint32_t)(j / S) & 1u;
        const int64_t b0 = u * p.P, b = b0 + pl;
        RegTile<float, MR, NR, Gm::PAIR> acc;
        acc.zero();
        ticket_wait(sm.ticket + 4 * s, j);
        bar_wait(sm.full + 8 * s, phase);
        {
            // the unit's spans start at these byte offsets inside the stage
            const uint32_t st = sm.ring + (uint32_t)(s * p.stage_bytes);
            const uint32_t misA = (uint32_t)(reinterpret_cast<uintptr_t>(p.A + b0 * sA * 4) & 15u);
            const uint32_t misB = (uint32_t)(reinterpret_cast<uintptr_t>(p.B + b0 * sB * 4) & 15u);
            const uint32_t pa = st + misA + (uint32_t)(pl * sA * 4);
            const uint32_t pb = st + (uint32_t)p.a_bytes + misB + (uint32_t)(pl * sB * 4);
            // k-step stride (bytes) of the MN-major operands
            const uint32_t ka = AK ? 4u : (uint32_t)lda * 4u, kb = BK ? 4u : (uint32_t)ldb * 4u;
            // fold this unit's stage addresses into the row / column registers
#pragma unroll
            for (int r = 0; r < (AK ? MR : 1); ++r) ra[r] += pa;
#pragma unroll
            for (int c = 0; c < (BK ? NR : 1); ++c) rb[c] += pb;
            // fragments of k-step k (da = k * ka, db = k * kb)
            auto frag = [&](float (&a)[MR], float (&bv)[NR], uint32_t da, uint32_t db) {
#pragma unroll
                for (int r = 0; r < MR; ++r) a[r] = lds32(AK ? ra[r] + da : ra[0] + da + (uint32_t)(LR * r * 4));
#pragma unroll
                for (int c = 0; c < NR; ++c) bv[c] = lds32(BK ? rb[c] + db : rb[0] + db + (uint32_t)(Gm::LC * c * 4));
            };
            // register double buffering (the paper's ping-pang):
            // k + 1's fragments load while k's FFMA2s issue -- for tiles of
            // <= 72 accumulators (the larger ones would spill at the 168-
            // register cap; they keep the plain unrolled loop)
            if constexpr (MR * NR > 72) {
#pragma unroll 4
                for (int k = 0; k < K; ++k) {
                    float a[MR], bv[NR];
                    frag(a, bv, (uint32_t)k * ka, (uint32_t)k * kb);
                    acc.rank1([&](int i) { return a[i]; }, [&](int j) { return bv[j]; });
                }
            } else {
                float a0[MR], b0[NR], a1[MR], b1[NR];
                frag(a0, b0, 0u, 0u);
                int k = 0;
                // both prefetches of an iteration stay below K; the last one
                // or two k-steps follow the loop (no load past the operand)
#pragma unroll 2
                for (; k + 2 < K; k += 2) {
                    frag(a1, b1, (uint32_t)(k + 1) * ka, (uint32_t)(k + 1) * kb);
                    acc.rank1([&](int i) { return a0[i]; }, [&](int j) { return b0[j]; });
                    frag(a0, b0, (uint32_t)(k + 2) * ka, (uint32_t)(k + 2) * kb);
                    acc.rank1([&](int i) { return a1[i]; }, [&](int j) { return b1[j]; });
                }
                if (k + 2 == K) {
                    frag(a1, b1, (uint32_t)(k + 1) * ka, (uint32_t)(k + 1) * kb);
                    acc.rank1([&](int i) { return a0[i]; }, [&](int j) { return b0[j]; });
                    acc.rank1([&](int i) { return a1[i]; }, [&](int j) { return b1[j]; });
                } else if (k < K) {
                    acc.rank1([&](int i) { return a0[i]; }, [&](int j) { return b0[j]; });
                }
            }
#pragma unroll
            for (int r = 0; r < (AK ? MR : 1); ++r) ra[r] -= pa;
#pragma unroll
            for (int c = 0; c < (BK ? NR : 1); ++c) rb[c] -= pb;
        }
        if (CS) {
            // fused epilogue in the stage's C span (C_in bulk-loaded with A
            // and B when beta != 0; the producer bulk-stores the span once
            // the group releases the stage)
            if (b < batch) {
                const uint32_t st = sm.ring + (uint32_t)(s * p.stage_bytes);
                const uint32_t misC = (uint32_t)(reinterpret_cast<uintptr_t>(p.C + b0 * sC * 4) & 15u);
                const uint32_t pc = st + (uint32_t)(p.a_bytes + p.b_bytes) + misC + (uint32_t)(pl * sC * 4);
#pragma unroll
                for (int c = 0; c < NR; ++c) {
                    const int col = C0 + Gm::col(tj, c);
#pragma unroll
                    for (int r = 0; r < MR; ++r) {
                        const int row = R0 + Gm::row(ti, r);
                        if (row < M && col < N) {
                            const uint32_t q = pc + (uint32_t)((col * ldc + row) * 4);
                            const float x = tile_at(acc, r, c);
                            sts32(q, beta_zero ? mul_rn(alpha, x) : fma_rn(alpha, x, mul_rn(beta, lds32(q))));
                        }
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            }
            __syncwarp();
            if (lane == 0) bar_arrive(sm.empty + 8 * s);
            continue;
        }
        __syncwarp();
        if (lane == 0) bar_arrive(sm.empty + 8 * s);
        if (b >= batch) continue;
        // fused epilogue, C through global: the C_in loads of a batch of
        // columns (<= 32 values) all issued before the batch's stores
        float v[MR][NR];
        acc.get(v);
        float *Cb = reinterpret_cast<float *>(p.C) + b * sC;
        constexpr int CB = (32 / MR) < 1 ? 1 : ((32 / MR) > NR ? NR : (32 / MR));
#pragma unroll
        for (int c0 = 0; c0 < NR; c0 += CB) {
            float ci[MR][CB];
            if (!beta_zero) {
#pragma unroll
                for (int cc = 0; cc < CB; ++cc) {
                    const int col = C0 + Gm::col(tj, c0 + cc);
#pragma unroll
                    for (int r = 0; r < MR; ++r) {
                        const int row = R0 + Gm::row(ti, r);
                        ci[r][cc] = (c0 + cc < NR && row < M && col < N) ? ldg_cs(Cb + (int64_t)col * ldc + row) : 0.f;
                    }
                }
            }
#pragma unroll
            for (int cc = 0; cc < CB; ++cc) {
                if (c0 + cc >= NR) break;
                const int col = C0 + Gm::col(tj, c0 + cc);
#pragma unroll
                for (int r = 0; r < MR; ++r) {
                    const int row = R0 + Gm::row(ti, r);
                    if (row < M && col < N)
                        stg_cs(Cb + (int64_t)col * ldc + row,
                               beta_zero ? mul_rn(alpha, v[r][c0 + cc])
                                         : fma_rn(alpha, v[r][c0 + cc], mul_rn(beta, ci[r][cc])));
                }
            }
        }
    }
}

__device__ __forceinline__ void bulk_load(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar, uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}

// Producer (slab staging): one thread streams the CTA's units in order
// j = 0, 1, ... (unit blockIdx.x * G + j % G + (j / G) * gridDim.x * G, the
// unit group j % G consumes) into the shared ring, stage j % S.
template <bool TA, bool TB, int G>
__device__ __forceinline__ void ksgs_producer(const IaatKsgParams &p, unsigned char *smem)
{
    const uint64_t pol = policy_evict_first();
    const SmemS sm(smem);
    const int64_t colsA = TA ? p.M : p.K, rowsA = TA ? p.K : p.M;
    const int64_t colsB = TB ? p.K : p.N, rowsB = TB ? p.N : p.K;
    const int S = p.S;
    // C span of the unit with sequence number j: elements [b0 * sC, (b0 + np) * sC)
    // (c_bytes != 0 only for ldc == M and packed problems: gap-free).  The
    // stage's C region holds it from its 16-byte-aligned start; the aligned
    // interior leaves by one bulk store, the <= 3 + 3 elements in the
    // granules shared with the neighbouring problems by plain stores.
    auto store_c = [&](int j, uint32_t creg) {
        const int64_t u = (int64_t)blockIdx.x * G + j % G + (int64_t)(j / G) * gridDim.x * G;
        const int64_t b0 = u * p.P;
        const int np = (int)min((int64_t)p.P, p.batch - b0);
        const uintptr_t a = reinterpret_cast<uintptr_t>(p.C + b0 * p.sC * 4);
        const uintptr_t e = a + (uintptr_t)((int64_t)np * p.sC * 4);
        const uintptr_t lo = a & ~(uintptr_t)15;
        const uintptr_t i0 = min((a + 15) & ~(uintptr_t)15, e), i1 = max(e & ~(uintptr_t)15, i0);
        for (uintptr_t x = a; x < i0; x += 4) stg_cs(reinterpret_cast<float *>(x), lds32(creg + (uint32_t)(x - lo)));
        for (uintptr_t x = i1; x < e; x += 4) stg_cs(reinterpret_cast<float *>(x), lds32(creg + (uint32_t)(x - lo)));
        if (i1 > i0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(i0),
                         "r"(creg + (uint32_t)(i0 - lo)), "r"((uint32_t)(i1 - i0))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    };
    int jn = 0;
    for (int j = 0;; ++j) {
        const int64_t u = (int64_t)blockIdx.x * G + j % G + (int64_t)(j / G) * gridDim.x * G;
        if (u >= p.nunits) break;
        const int64_t b0 = u * p.P;
        const int np = (int)min((int64_t)p.P, p.batch - b0);
        // the 16-byte-aligned span enclosing the unit's bytes of one operand
        // (over-read <= 15 B per end, inside granules that hold valid data)
        auto span = [](const char *base, int64_t first, int64_t stride, int np_, int64_t rows, int64_t cols,
                       int64_t ld, uintptr_t &lo) {
            const uintptr_t a = reinterpret_cast<uintptr_t>(base + first * stride * 4);
            const uintptr_t e = a + (uintptr_t)(((int64_t)(np_ - 1) * stride + (cols - 1) * ld + rows) * 4);
            lo = a & ~(uintptr_t)15;
            return (uint32_t)(((e + 15) & ~(uintptr_t)15) - lo);
        };
        uintptr_t loA, loB;
        const uint32_t nA = span(p.A, b0, p.sA, np, rowsA, colsA, p.lda, loA);
        const uint32_t nB = span(p.B, b0, p.sB, np, rowsB, colsB, p.ldb, loB);
        const int s = j % S;
        if (j >= S) bar_wait(sm.empty + 8 * s, (uint32_t)(j / S - 1) & 1u);
        const uint32_t st = sm.ring + (uint32_t)(s * p.stage_bytes), fb = sm.full + 8 * s;
        if (p.c_bytes && j >= S) store_c(j - S, st + (uint32_t)(p.a_bytes + p.b_bytes));
        ticket_set(sm.ticket + 4 * s, j);
        uintptr_t loC = 0;
        const uint32_t nC = p.beta_zero ? 0u : span(p.C, b0, p.sC, np, p.M, p.N, p.ldc, loC);
        bar_expect_tx(fb, nA + nB + (p.c_bytes ? nC : 0u));
        bulk_load(st, reinterpret_cast<const void *>(loA), nA, fb, pol);
        bulk_load(st + (uint32_t)p.a_bytes, reinterpret_cast<const void *>(loB), nB, fb, pol);
        if (p.c_bytes) {
            if (nC) {
                // the span store of the stage's previous unit must have read
                // its C region before C_in lands there
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                bulk_load(st + (uint32_t)(p.a_bytes + p.b_bytes), reinterpret_cast<const void *>(loC), nC, fb, pol);
            }
        } else if (nC) {
            bulk_prefetch_l2(reinterpret_cast<const void *>(loC), nC);
        }
        ++jn;
    }
    if (p.c_bytes) {
        // the last S units: store each C span once its group is done
        for (int j = max(0, jn - S); j < jn; ++j) {
            const int s = j % S;
            bar_wait(sm.empty + 8 * s, (uint32_t)(j / S) & 1u);
            store_c(j, sm.ring + (uint32_t)(s * p.stage_bytes + p.a_bytes + p.b_bytes));
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

// CS: C through the stage (p.c_bytes != 0; the launcher picks the instance)
template <bool TA, bool TB, int MR, int NR, int LR, int G, int W, bool CS>
__device__ __forceinline__ void ksgs_body(const IaatKsgParams &p)
{
    static_assert(G * W == 8 || G * W == 12, "ksgs: two or three warpgroups of consumers");
    extern __shared__ __align__(1024) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        const SmemS sm(smem);
        for (int s = 0; s < p.S; ++s) {
            bar_init(sm.full + 8 * s, 1);
            bar_init(sm.empty + 8 * s, W);
            ticket_set(sm.ticket + 4 * s, -1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(IAAT_KSG_PRODUCER_REGS));
        if (threadIdx.x == 0) ksgs_producer<TA, TB, G>(p, smem);
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(IAAT_KSG_CONSUMER_REGS_OF(G * W)));
        const int c = warp - 4;
        ksgs_consumer<TA, TB, MR, NR, LR, G, W, CS>(p, smem, c / W, c % W, lane);
    }
}

}  // namespace ksg
}  // namespace iaat
