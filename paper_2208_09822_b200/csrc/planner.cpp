// planner.cpp -- the run-time stage (Sec. III-B, V).
//
// The paper's input-aware adaptive tile algorithm tiles C into blocks that
// each have the exact size of a generated kernel, guided by
// three principles: bigger blocks, minimal memops
// ((m_0+n_0+...+m_a+n_a)K + 2mn elements moved into registers) and SIMD
// friendliness (the contiguous block dimension a multiple of the vector
// length).  On B200 the same decision is made per call, then cached:
//
//  (i)   an EXACT decomposition of M (and N) into at most two strips of
//        catalog tile sizes (Alg. 2's m[] / n[] arrays of (dim, nums) pairs,
//        PAPER.md:261-262, 319), strips whose size is a multiple of the 16-byte
//        vector first (SIMD friendly);
//  (ii)  the tile classes = strip products (blocksC), each run
//        by its own warps (warp-uniform, no predicated edge code);
//  (iii) P problems per pipeline stage, S stages and the persistent grid,
//        chosen by a small cost model of one SM: HBM bytes of a group vs the
//        issue cycles of its tiles (including idle lanes), plus the wave
//        quantisation of the whole call;
//  (iv)  the staging mode (one slab copy vs per-problem copies) and whether
//        the 16-byte vector paths are legal (alignment of every address).
// Ties go to fewer memops (the paper's cost), then bigger tiles.
#include "planner.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "gen/catalog.inc"

namespace iaat {

namespace {

constexpr double kHbmBytesPerClk = 22.0;  // 6.5 TB/s / 148 SMs / ~2.0 GHz
constexpr double kDfmaPerClk = 64.0;      // fp64 FMA lanes per SM per clock
constexpr double kGroupOverhead = 150.0;  // mbarrier round trip + dispatch per group

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct DimSplit {
    Strip s[2];
    int n = 0;
    int tiles() const { return s[0].count + (n > 1 ? s[1].count : 0); }
    bool operator==(const DimSplit &o) const
    {
        if (n != o.n) return false;
        for (int i = 0; i < n; ++i)
            if (s[i].size != o.s[i].size || s[i].count != o.s[i].count) return false;
        return true;
    }
};

// Order strips: sizes that are multiples of the vector width first, so every
// vector-capable tile starts on a vector boundary; then larger first.
void order(DimSplit &d, int vw)
{
    if (d.n < 2) return;
    bool a = d.s[0].size % vw == 0, b = d.s[1].size % vw == 0;
    if ((!a && b) || (a == b && d.s[1].size > d.s[0].size)) std::swap(d.s[0], d.s[1]);
}

void push_unique(std::vector<DimSplit> &v, DimSplit d, int vw)
{
    if (d.n == 2 && d.s[1].count == 0) d.n = 1;
    if (d.n == 2 && d.s[0].count == 0) {
        d.s[0] = d.s[1];
        d.n = 1;
    }
    if (d.n == 2 && d.s[0].size == d.s[1].size) {
        d.s[0].count += d.s[1].count;
        d.n = 1;
    }
    order(d, vw);
    for (auto &e : v)
        if (e == d) return;
    v.push_back(d);
}

// 1-D exact decompositions of D into at most two tile sizes <= maxt:
// greedy largest-first (TileSingleDim) and balanced ("average
// the last two pieces").
std::vector<DimSplit> splits(int D, int maxt, int vw)
{
    std::vector<DimSplit> v;
    for (int t = 1; t <= std::min(D, maxt); ++t) {
        DimSplit g;
        g.s[0] = {t, D / t};
        g.n = 1;
        if (D % t) {
            g.s[1] = {D % t, 1};
            g.n = 2;
        }
        push_unique(v, g, vw);
        int c = (D + t - 1) / t;
        DimSplit b;
        b.s[0] = {D / c + 1, D % c};
        b.s[1] = {D / c, c - D % c};
        b.n = 2;
        push_unique(v, b, vw);
    }
    return v;
}

struct Geo {
    int64_t spanA, spanB;  // bytes of one problem's operand span
    int elt;
};

struct Candidate {
    bool ok = false;
    double total = 1e300;
    double group = 0;
    int64_t memops = 0;
    int area = 0;
    int P = 0, S = 0, W = 0;
    int family = IAAT_FAM_FMA;
    DimSplit ms, ns;
    int wm = 1, wn = 1;  // DMMA warp tile (in 8x8 blocks)
    int capA = 0, capB = 0, slotA = 0, slotB = 0, modeA = 0, modeB = 0;
    IaatClass cls[IAAT_MAX_CLASSES];
    int ncls = 0;
};

// Staging layout for one operand at P problems per group.
void stage_layout(int64_t span, int64_t stride_b, int P, bool ptr_array, int &mode, int &slot, int &cap)
{
    const int64_t slab = (int64_t)(P - 1) * std::llabs(stride_b) + span;
    if (!ptr_array && (P == 1 || slab * 4 <= (int64_t)P * span * 5)) {
        mode = IAAT_STAGE_SLAB;
        slot = 0;
        cap = (int)round_up(slab + 32, 128);
    } else {
        mode = IAAT_STAGE_PERPROB;
        slot = (int)round_up(span + 32, 16);
        cap = (int)round_up((int64_t)P * slot, 128);
    }
}

bool better(const Candidate &a, const Candidate &b)
{
    if (!a.ok) return false;
    if (!b.ok) return true;
    if (a.total < b.total * 0.995) return true;
    if (b.total < a.total * 0.995) return false;
    if (a.memops != b.memops) return a.memops < b.memops;
    return a.area > b.area;
}

// Thread instructions of one FMA tile over the whole K (model).
double fma_tile_instr(const PlanRequest &r, bool vec, int mr, int nr, int vw)
{
    const bool a_kc = r.transA == 1, b_kc = r.transB == 0;
    auto loads = [&](bool kcontig, int d) -> double {
        if (!vec) return d;
        if (kcontig) return (double)d / vw;  // one vector per row per vw k-steps
        return d % vw == 0 ? (double)d / vw : d;
    };
    const double per_k = mr * nr + loads(a_kc, mr) + loads(b_kc, nr) + 0.5;
    const double epi = mr * nr * (r.beta_zero ? 2.0 : 4.0);
    return r.K * per_k + epi + 40.0;
}

}  // namespace

bool catalog_has(int dtype, int trans_idx, int family, int mr, int nr)
{
    for (const auto &e : kCatalog)
        if (e.family == family && e.dtype == dtype && e.trans == trans_idx && e.mr == mr && e.nr == nr)
            return true;
    return false;
}

int catalog_code(int family, int mr, int nr)
{
    return family == IAAT_FAM_FMA ? IAAT_FMA_CODE(mr, nr) : IAAT_DMMA_CODE(mr / 8, nr / 8);
}

const char *catalog_json() { return kCatalogJson; }

Plan make_plan(const PlanRequest &r)
{
    Plan plan;
    const int elt = r.dtype == 0 ? 4 : 8;
    const int vw = 16 / elt;
    const int tidx = r.transA * 2 + r.transB;
    const int64_t M = r.M, N = r.N, K = r.K;
    Geo geo;
    geo.elt = elt;
    // stored shapes (reading A1)
    const int64_t colsA = r.transA ? M : K, rowsA = r.transA ? K : M;
    const int64_t colsB = r.transB ? K : N, rowsB = r.transB ? N : K;
    geo.spanA = ((colsA - 1) * r.lda + rowsA) * elt;
    geo.spanB = ((colsB - 1) * r.ldb + rowsB) * elt;

    // 16-byte vector paths are legal iff every problem's A, B, C base and
    // every column start is 16 B aligned (strided API only).
    auto al16 = [&](int64_t el) { return (el * elt) % 16 == 0; };
    const bool vec = !r.ptr_array && r.align % 16 == 0 && al16(r.lda) && al16(r.ldb) && al16(r.ldc) &&
                     (r.batch <= 1 || (al16(r.sA) && al16(r.sB) && al16(r.sC)));
    plan.vec = vec ? 1 : 0;

    const double hbm_per_problem =
        (double)(M * K + K * N + M * N * (r.beta_zero ? 1 : 2)) * elt;
    const int64_t sAb = r.sA * elt, sBb = r.sB * elt;
    const int smem_avail = IAAT_SMEM_LIMIT - IAAT_BAR_BYTES;

    Candidate best;

    auto finish_candidate = [&](Candidate &c, double issue_per_group, double pipe_per_group, int P) {
        // smem / stages
        stage_layout(geo.spanA, sAb, P, r.ptr_array, c.modeA, c.slotA, c.capA);
        stage_layout(geo.spanB, sBb, P, r.ptr_array, c.modeB, c.slotB, c.capB);
        const int64_t stage = (int64_t)c.capA + c.capB;
        int S = (int)std::min<int64_t>(4, smem_avail / stage);
        if (S < 1) return false;
        if (S < 2 && P > 1) return false;
        c.S = S;
        c.P = P;
        const double mem = hbm_per_problem * P / kHbmBytesPerClk;
        double grp = std::max(mem, std::max(issue_per_group, pipe_per_group)) + kGroupOverhead;
        if (S == 1) grp = mem + std::max(issue_per_group, pipe_per_group) + kGroupOverhead;
        const int64_t ngroups = (r.batch + P - 1) / P;
        const int64_t grid = std::min<int64_t>(ngroups, r.sm_count);
        const int64_t waves = (ngroups + grid - 1) / grid;
        c.group = grp;
        c.total = grp * (double)waves + 2000.0;  // + launch / pipeline fill
        c.ok = true;
        return true;
    };

    // ------------------------------------------------------------ FMA family
    const int maxt = 8;
    auto msplits = splits((int)M, maxt, vw);
    auto nsplits = splits((int)N, maxt, vw);
    for (const auto &ms : msplits) {
        for (const auto &ns : nsplits) {
            // classes and catalog availability
            bool avail = true;
            int64_t memops = 2 * M * N;
            int area = 0;
            struct C4 { int mr, nr, tiles, tm, rb, cb; double instr; } cl[4];
            int ncl = 0;
            int rb = 0;
            for (int a = 0; a < ms.n; ++a) {
                int cb = 0;
                for (int b = 0; b < ns.n; ++b) {
                    const int mr = ms.s[a].size, nr = ns.s[b].size;
                    if (!catalog_has(r.dtype, tidx, IAAT_FAM_FMA, mr, nr)) avail = false;
                    const int tiles = ms.s[a].count * ns.s[b].count;
                    cl[ncl++] = {mr, nr, tiles, ms.s[a].count, rb, cb,
                                 fma_tile_instr(r, vec, mr, nr, vw)};
                    memops += (int64_t)tiles * (mr + nr) * K;
                    area = std::max(area, mr * nr);
                    cb += ns.s[b].size * ns.s[b].count;
                }
                rb += ms.s[a].size * ms.s[a].count;
            }
            if (!avail) continue;
            const int tiles_pp = ms.tiles() * ns.tiles();
            const int64_t pmax_batch = std::max<int64_t>(1, (r.batch + r.sm_count - 1) / r.sm_count);
            for (int P = 1; P <= 512; ++P) {
                if (P > pmax_batch && P > 1) break;
                int W = 0;
                double issue = 0;
                for (int q = 0; q < ncl; ++q) {
                    const int w = (P * cl[q].tiles + 31) / 32;
                    W += w;
                    issue += w * cl[q].instr;
                }
                if (W > IAAT_MAX_COMPUTE_WARPS) break;
                (void)tiles_pp;
                const double rate = std::min(3.5, 0.5 * W);
                double pipe = 0;
                if (r.dtype == 1) pipe = (double)P * M * N * K / kDfmaPerClk;
                Candidate c;
                c.family = IAAT_FAM_FMA;
                c.ms = ms;
                c.ns = ns;
                c.memops = memops;
                c.area = area;
                c.W = W;
                if (!finish_candidate(c, issue / rate, pipe, P)) continue;
                // classes
                int wb = 0;
                c.ncls = ncl;
                for (int q = 0; q < ncl; ++q) {
                    const int w = (P * cl[q].tiles + 31) / 32;
                    c.cls[q] = IaatClass{catalog_code(IAAT_FAM_FMA, cl[q].mr, cl[q].nr), wb, wb + w,
                                         cl[q].tiles, cl[q].tm, cl[q].rb, cl[q].mr, cl[q].cb,
                                         cl[q].nr, cl[q].tiles};
                    wb += w;
                }
                if (better(c, best)) best = c;
            }
        }
    }

    // ------------------------------------------------------------ DMMA family (fp64)
    if (r.dtype == 1 && M % 8 == 0 && N % 8 == 0) {
        for (int wm = 1; wm <= 2; ++wm)
            for (int wn = 1; wn <= 2; ++wn) {
                if ((M / 8) % wm || (N / 8) % wn) continue;
                if (!catalog_has(1, tidx, IAAT_FAM_DMMA, 8 * wm, 8 * wn)) continue;
                const int tm = (int)(M / (8 * wm)), tn = (int)(N / (8 * wn));
                const int tiles = tm * tn;
                const int64_t memops = (int64_t)tiles * (8 * wm + 8 * wn) * K + 2 * M * N;
                const int64_t pmax_batch = std::max<int64_t>(1, (r.batch + r.sm_count - 1) / r.sm_count);
                // per item (one warp tile over K): DMMAs + fragment loads + epilogue
                const double kst = (double)((K + 3) / 4);
                const double instr_item = kst * (wm * wn + wm + wn + 2) + wm * wn * (r.beta_zero ? 6 : 10) + 30;
                for (int P = 1; P <= 64; ++P) {
                    if (P > pmax_batch && P > 1) break;
                    const int items = P * tiles;
                    for (int W = 4; W <= IAAT_MAX_COMPUTE_WARPS; W += 1) {
                        if (W > items && W > 4) break;
                        const double per_warp_items = std::ceil((double)items / W);
                        const double issue = per_warp_items * W * instr_item / std::min(3.5, 0.5 * W);
                        // DMMA pipe: 128 flop / clk / SM at the fp64 peak
                        const double pipe = (double)P * 2.0 * M * N * K / 128.0 *
                                            (per_warp_items * W / items);
                        Candidate c;
                        c.family = IAAT_FAM_DMMA;
                        c.ms.s[0] = {8 * wm, tm};
                        c.ms.n = 1;
                        c.ns.s[0] = {8 * wn, tn};
                        c.ns.n = 1;
                        c.wm = wm;
                        c.wn = wn;
                        c.memops = memops;
                        c.area = 64 * wm * wn;
                        c.W = W;
                        if (!finish_candidate(c, issue, pipe, P)) continue;
                        c.ncls = 1;
                        c.cls[0] = IaatClass{catalog_code(IAAT_FAM_DMMA, 8 * wm, 8 * wn), 0, W, tiles, tm,
                                             0, 8 * wm, 0, 8 * wn, tiles};
                        if (better(c, best)) best = c;
                    }
                }
            }
    }

    if (!best.ok) {
        plan.status = 5;  // IAAT_ERROR_NOT_SUPPORTED
        return plan;
    }
    IaatKParams &kp = plan.kp;
    std::memset(&kp, 0, sizeof(kp));
    kp.sA = r.sA;
    kp.sB = r.sB;
    kp.sC = r.sC;
    kp.batch = r.batch;
    kp.ngroups = (r.batch + best.P - 1) / best.P;
    kp.M = (int)M;
    kp.N = (int)N;
    kp.K = (int)K;
    kp.lda = (int)r.lda;
    kp.ldb = (int)r.ldb;
    kp.ldc = (int)r.ldc;
    kp.P = best.P;
    kp.S = best.S;
    kp.n_compute_warps = best.W;
    kp.modeA = best.modeA;
    kp.modeB = best.modeB;
    kp.spanA = (int)geo.spanA;
    kp.spanB = (int)geo.spanB;
    kp.slotA = best.slotA;
    kp.slotB = best.slotB;
    kp.capA = best.capA;
    kp.capB = best.capB;
    kp.stage_bytes = best.capA + best.capB;
    kp.beta_zero = r.beta_zero;
    kp.prefetch_c = r.beta_zero ? 0 : 1;
    kp.nclasses = best.ncls;
    for (int q = 0; q < best.ncls; ++q) kp.cls[q] = best.cls[q];
    plan.family = best.family;
    plan.grid = (int)std::min<int64_t>(kp.ngroups, r.sm_count);
    plan.block = (best.W + 1) * 32;
    plan.smem = IAAT_BAR_BYTES + best.S * kp.stage_bytes;
    plan.nm = best.ms.n;
    plan.nn = best.ns.n;
    for (int i = 0; i < 2; ++i) {
        plan.mstrip[i] = best.ms.s[i];
        plan.nstrip[i] = best.ns.s[i];
    }
    plan.memops = best.memops;
    plan.est_cycles = best.group;
    plan.est_total = best.total;
    plan.status = 0;
    return plan;
}

std::string plan_json(const PlanRequest &r, const Plan &p)
{
    char buf[512];
    std::string s = "{";
    auto add = [&](const char *fmt, auto... a) {
        std::snprintf(buf, sizeof buf, fmt, a...);
        s += buf;
    };
    add("\"status\": %d, \"dtype\": \"%s\", \"trans\": \"%c%c\", \"M\": %lld, \"N\": %lld, \"K\": %lld, ",
        p.status, r.dtype ? "f64" : "f32", r.transA ? 'T' : 'N', r.transB ? 'T' : 'N', (long long)r.M,
        (long long)r.N, (long long)r.K);
    if (p.status != 0) {
        s += "\"classes\": []}";
        return s;
    }
    const IaatKParams &k = p.kp;
    add("\"family\": \"%s\", \"vec\": %d, \"P\": %d, \"S\": %d, \"compute_warps\": %d, \"grid\": %d, "
        "\"block\": %d, \"smem\": %d, \"ngroups\": %lld, ",
        p.family == IAAT_FAM_DMMA ? "dmma" : "fma", p.vec, k.P, k.S, k.n_compute_warps, p.grid, p.block,
        p.smem, (long long)k.ngroups);
    add("\"stage_a\": \"%s\", \"stage_b\": \"%s\", \"cap_a\": %d, \"cap_b\": %d, \"prefetch_c\": %d, ",
        k.modeA ? "perprob" : "slab", k.modeB ? "perprob" : "slab", k.capA, k.capB, k.prefetch_c);
    add("\"m_strips\": [");
    for (int i = 0; i < p.nm; ++i) add("%s[%d, %d]", i ? ", " : "", p.mstrip[i].size, p.mstrip[i].count);
    add("], \"n_strips\": [");
    for (int i = 0; i < p.nn; ++i) add("%s[%d, %d]", i ? ", " : "", p.nstrip[i].size, p.nstrip[i].count);
    add("], \"memops\": %lld, \"est_cycles_per_group\": %.1f, \"est_cycles_total\": %.1f, \"classes\": [",
        (long long)p.memops, p.est_cycles, p.est_total);
    for (int q = 0; q < k.nclasses; ++q) {
        const IaatClass &c = k.cls[q];
        add("%s{\"code\": %d, \"mr\": %d, \"nr\": %d, \"tiles\": %d, \"tm\": %d, \"row_base\": %d, "
            "\"col_base\": %d, \"warp_begin\": %d, \"warp_end\": %d}",
            q ? ", " : "", c.code, c.mr, c.nr, c.tiles, c.tm, c.row_base, c.col_base, c.warp_begin,
            c.warp_end);
    }
    s += "]}";
    return s;
}

}  // namespace iaat
