// planner.h -- run-time stage: input-aware planning of one batched call
// (Sec. III-B / V).
#pragma once
#include <stdint.h>

#include <string>

#include "iaat_params.h"

namespace iaat {

struct PlanRequest {
    int dtype;          // 0 fp32, 1 fp64
    int transA, transB; // 0 = N, 1 = T
    int64_t M, N, K;
    int64_t lda, ldb, ldc;
    int64_t sA, sB, sC; // strides (elements); ignored for the pointer-array API
    int64_t batch;
    int beta_zero, alpha_zero;
    int64_t align;      // common alignment (bytes) of the A/B/C base addresses
    int sm_count;
    int ptr_array;      // 1 = iaat_gemm_batched
};

// One strip of a 1-D decomposition (Alg. 2's (dim, nums) pairs).
struct Strip {
    int size;
    int count;
};

// Geometry of one operand's 3-D TMA tensor map (K-streamed family); the
// base address is bound at call time.
struct TmaGeo {
    uint64_t dim[3];      // elements: stored rows, stored cols, batch
    uint64_t stride[2];   // bytes: ld * elt, problem stride * elt
    uint32_t box[3];      // box extents (elements)
    int swizzle128;       // 1: CU_TENSOR_MAP_SWIZZLE_128B (K-major operand)
    int swizzle64;        // 1: CU_TENSOR_MAP_SWIZZLE_64B (K-major operand, 16-element K-chunks)
};

struct Plan {
    int status = 0;        // iaat_status_t (SUCCESS or NOT_SUPPORTED)
    IaatKParams kp{};      // pointers / alpha / beta filled at call time
    int ks = 0;            // 1: K-streamed family (ksp + tmA/tmB are the plan)
    int single = 0;        // K-streamed: 1 = a single-class kernel (tile ksp.cls[0].mr x nr)
    int ksd = 0;           // K-streamed: 1 = fp64 DMMA warp-tile kernel (iaat_ksd_*)
    IaatKsParams ksp{};
    TmaGeo tmA{}, tmB{};
    int ksg = 0;           // 1: ksg family (kgp + tmA/tmB/tmC, kernel kKsgCatalog[kg_entry])
                           // 2: ksgs -- slab-staged lane grids (kgp only, kernel kKsgsCatalog[kg_entry])
    int kg_entry = -1;
    IaatKsgParams kgp{};
    TmaGeo tmC{};
    int grid = 0, block = 0, smem = 0;
    int vec = 0;           // kernel variant: 16-byte vector paths enabled
    int family = 0;        // IAAT_FAM_FMA or IAAT_FAM_DMMA
    int ctas = 1;          // resident CTAs per SM the plan is sized for
    int tuned = 0;         // 1: knobs came from the install-time tuning table
    Strip mstrip[2]{}, nstrip[2]{};
    int nm = 0, nn = 0;    // strips used per dimension
    int64_t memops = 0;    // paper cost: sum_i (m_i + n_i) K + 2 M N
    double est_cycles = 0; // modelled SM cycles per group
    double est_total = 0;  // modelled cycles for the whole call
};

// Build the plan (pure host function; no CUDA calls).
Plan make_plan(const PlanRequest &r);

// JSON description (iaat_plan_describe).
std::string plan_json(const PlanRequest &r, const Plan &p);

// True if (dtype, trans, family, mr, nr) is in the install-time catalog.
bool catalog_has(int dtype, int trans_idx, int family, int mr, int nr);
int catalog_code(int family, int mr, int nr);
const char *catalog_json();

// Paper-faithful tiling of an SGEMM_NN M x N block with the Table I catalog
// (SURVEY f3): mode 0 = Alg. 2 literal, 1 = optimal DP; JSON.
std::string paper_tile_json(int mode, int M, int N);

}  // namespace iaat
