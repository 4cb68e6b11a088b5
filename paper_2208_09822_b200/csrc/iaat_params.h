// iaat_params.h -- the "kernel executing plan" (Sec. V-B)
// as it crosses the host->device boundary: one POD struct passed by value
// (__grid_constant__) to the single persistent launch of a call.
//
// Host (planner.cpp, api.cu) and device (iaat_device.cuh) both include this.
#pragma once
#include <stdint.h>

#define IAAT_MAX_CLASSES 4
#define IAAT_MAX_STAGES 6
#define IAAT_MAX_THREADS 512          // __launch_bounds__ of every pipeline kernel
#define IAAT_MAX_COMPUTE_WARPS 15     // + 1 producer warp
#define IAAT_SMEM_LIMIT (227 * 1024)  // opt-in dynamic shared memory per CTA
#define IAAT_BAR_BYTES 128            // mbarriers live in the first 128 B

// Staging modes for an operand.
enum IaatStage : int {
    IAAT_STAGE_SLAB = 0,     // one bulk copy of the enclosing 16 B-aligned span of P problems
    IAAT_STAGE_PERPROB = 1,  // one bulk copy per problem into its own smem slot
};

// Micro-tile families of the install-time catalog.
enum IaatFamily : int {
    IAAT_FAM_FMA = 0,     // per-thread mr x nr FFMA/DFMA register tile (slab staging)
    IAAT_FAM_DMMA = 1,    // per-warp (8*wm) x (8*wn) DMMA.8x8x4 tile (fp64 only, slab staging)
    IAAT_FAM_KS_FMA = 2,  // FMA tiles, K-streamed TMA staging (iaat_ks.cuh)
    IAAT_FAM_KS_DMMA = 3, // DMMA warp tiles, K-streamed TMA staging (fp64 only)
    IAAT_FAM_KS1_FMA = 4, // single-class K-streamed kernels (one per tile; the big tiles)
    IAAT_FAM_KSU_FMA = 6, // single-class K-streamed fp32, uniform swizzle phase only (tm/tn % 8 == 0)
    IAAT_FAM_KSG = 7,     // fp32 lane-grid register tiles, warp groups, C through smem (iaat_ksg.cuh)
    IAAT_FAM_KSGS = 8,    // the same lane grids on slab staging, any alignment (iaat_ksg.cuh ksgs_*)
};

// One tile class: all tiles of one exact size (mr x nr) inside one row strip
// and one column strip of C (Alg. 2 "blocksC", "m[]", "n[]").
// Warps [warp_begin, warp_end) run it; lane index -> (problem, tile).
struct IaatClass {
    int code;        // catalog entry (dispatch switch case), see catalog.inc
    int warp_begin;  // first compute warp of this class
    int warp_end;    // one past the last
    int tiles;       // tiles of this class per problem (= tm * tn)
    int tm;          // tiles along M inside the class (row-fastest tile order)
    int row_base;    // first row of the class' row strip
    int mr;          // tile rows (== the catalog entry's MR; kept for host printing)
    int col_base;    // first column of the class' column strip
    int nr;          // tile columns
    int tn;          // tiles along N inside the class
    int colfast;     // linear lane/tile order: 0 = row tiles fastest, 1 = column tiles fastest
    int bm;          // 0: linear mapping (a warp may span problems);  >0: blocked mapping --
                     // each warp owns a bm x (32/bm) block of tiles of ONE problem
};

struct IaatKParams {
    // strided API: byte base pointers; pointer-array API: the arrays (else null)
    const char *A;
    const char *B;
    char *C;
    const void *const *Aarr;
    const void *const *Barr;
    void *const *Carr;
    int64_t sA, sB, sC;  // strides in elements (strided API)
    int64_t batch;       // problems in this call
    int64_t ngroups;     // ceil(batch / P)
    double alpha, beta;
    double alpha_i, beta_i;  // imaginary parts (complex dtypes; 0 otherwise)
    int M, N, K;
    int lda, ldb, ldc;
    int P;               // problems per group (one pipeline stage)
    int S;               // pipeline stages
    int n_compute_warps;
    int modeA, modeB, modeC;  // IaatStage
    int spanA, spanB, spanC;  // bytes spanned by one problem's A / B / C
    int slotA, slotB, slotC;  // per-problem smem slot (PERPROB mode), bytes
    int capA, capB, capC;     // smem bytes reserved per stage (multiples of 128); capC = 0: C_in not staged
    int stage_bytes;          // capA + capB + capC
    int beta_zero;            // 1: C is write-only
    int c_in_smem;            // 1: C_in staged with A/B (beta != 0); 0 and beta != 0: read from global
    int prefetch_c;           // 1: producer prefetches the C span into L2 (when C_in is read from global)
    int nclasses;
    IaatClass cls[IAAT_MAX_CLASSES];
};

// ---------------------------------------------------------------- K-streamed family
// Kernel executing plan of the "ks" kernels (iaat_ks.cuh): units of P
// consecutive problems, streamed in K-chunks of kc elements through an
// S-stage ring of TMA boxes.  The two CUtensorMaps travel as separate
// __grid_constant__ kernel parameters.
#define IAAT_KS_MAX_STAGES 12
// fp64 / ZGEMM DMMA warp tiles of 10 or more 8x8 blocks keep their
// accumulators without spills only above 128 registers per thread: their
// kernels are compiled for at most 384 threads (168 registers) and the
// planner sizes their CTAs accordingly (spill-free catalog).
#define IAAT_KSD_THREADS(wm, wn) ((wm) * (wn) >= 10 ? 384 : IAAT_MAX_THREADS)
#define IAAT_KS_BAR_BYTES 256   // mbarriers; the stage ring starts at the next 1024 B boundary

struct IaatKsParams {
    char *C;
    int64_t sC;          // C stride (elements)
    int64_t batch;
    int64_t nunits;      // ceil(batch / P)
    double alpha, beta;
    int M, N, K, ldc;
    int P, S, kc, nchunks;
    int n_compute_warps;
    int a_pitch, b_pitch;  // MN-major operands: smem row pitch (elements) = TMA box inner dim
    int a_bytes, b_bytes;  // smem bytes of one stage's A / B region (multiples of 1024)
    int a_tx, b_tx;        // bytes one TMA box of A / B delivers (the full box)
    int stage_bytes;       // a_bytes + b_bytes
    int beta_zero;
    int c_vec;             // 16-byte C accesses legal (C base, ldc, stride aligned)
    int debug;             // measurement only (IAAT_DEBUG_KS): bit0 skip the k loop, bit1 skip the epilogue, bit2 do not wait for data (timing only)
    // LDGSTS staging (ldgsts = 1): inputs whose ld / stride / base break the
    // TMA 16-byte rules are copied element-wise with cp.async (any element
    // alignment) into the SAME smem layouts the TMA boxes produce
    int ldgsts;
    int cplx;              // 1: complex fp64 (ZGEMM) DMMA kernels -- TMA boxes over the real (re, im) view
    int c_elt;             // bytes per C element (sizeof(T), or 16 for complex fp64)
    double alpha_i, beta_i;
    const char *A, *B;     // base pointers (LDGSTS mode)
    int64_t sA, sB;        // problem strides (elements)
    int lda, ldb;
    int nclasses;
    IaatClass cls[IAAT_MAX_CLASSES];
};

// ---------------------------------------------------------------- K-streamed group family
// Kernel executing plan of the "ksg" kernels (iaat_ksg.cuh): fp32, one
// lane-grid tile class over an Mv x Nv "virtual" problem (Mv >= M, Nv >= N;
// rows / columns past M / N are the copy engine's zero fill and are never
// stored), G warp groups of W consumer warps (+ one producer warp per
// group), each group with its own S-stage ring of K-chunks, its own C
// buffer and every G-th unit of P problems.
#define IAAT_KSG_MAX_STAGES 8
#define IAAT_KSG_MAX_GROUPS 4
#define IAAT_KSG_GROUP_BARS (2 * IAAT_KSG_MAX_STAGES + 2)  // full[S], empty[S], cfull, cready
#define IAAT_KSG_BAR_BYTES 1024
#define IAAT_KSGS_MAX_STAGES 32  // ksgs: one shared ring; full[], empty[], ticket[] in the 1 KB barrier area

struct IaatKsgParams {
    int64_t batch;
    int64_t nunits;        // ceil(batch / P)
    double alpha, beta;
    int M, N, K;           // the problem
    int Mv, Nv;            // the tiled (virtual) extent: Mv - M, Nv - N rows / columns of zero fill
    int P, S, nchunks;     // problems per unit, stages per group ring (ksgs: of the one shared ring), ceil(K / KC)
    int a_pitch, b_pitch;  // MN-major operands: smem row pitch (elements) = TMA box inner dim
    int c_pitch;           // C buffer: elements per column (TMA box inner dim >= Mv; padded against bank conflicts)
    int a_bytes, b_bytes;  // smem bytes of one stage's A / B region (multiples of 1024)
    int a_tx, b_tx;        // bytes one TMA box of A / B delivers (the full box, zero fill included)
    int stage_bytes;       // a_bytes + b_bytes
    int c_bytes;           // smem bytes of the group's C buffer (box [P][Nv][c_pitch], multiple of 1024)
    int c_tx;              // bytes one TMA box of C delivers
    int group_bytes;       // S * stage_bytes + c_bytes (one group's ring + C buffer)
    int beta_zero;
    int bm;                // warp blocks along Mv per problem
    int wpp;               // warp blocks per problem (bm * blocks along Nv)
    // column-pair boxes (pairv = 1; kernel instances PV): packed operands
    // whose ld's are even but not multiples of 4 (n = 2 mod 4: 8-byte, not
    // 16-byte, column pitches) seen as tensors of column PAIRS -- rows of
    // 2 * ld elements, a legal 16-byte TMA stride.  MN-major operands and C
    // land exactly as before with pitch ld (= rows; 8-byte vector accesses);
    // a K-major operand lands as two unswizzled boxes per K-chunk, even
    // columns then odd columns (a_half / b_half bytes apart), rows of
    // kc + 4 elements.  Rows past M of a warp block read the next column and
    // are never stored.
    int pairv;
    int a_half, b_half;
    // slab staging (kernels iaat_ksgs_*): for inputs the TMA rules exclude
    // (ld's / strides / bases not 16-byte aligned).  Each stage holds the P
    // problems of a unit verbatim -- one cp.async.bulk per operand of the
    // 16-byte-aligned span enclosing them -- and C goes through global.
    const char *A, *B;
    char *C;
    int64_t sA, sB, sC;    // problem strides (elements; packed: sA = lda * cols of A)
    int lda, ldb, ldc;
};
