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

#include <dlfcn.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "gen/catalog.inc"

namespace iaat {

namespace {

// element bytes of a dtype: 0 fp32, 1 fp64, 2 complex fp32, 3 complex fp64
int elt_of(int dtype) { return dtype == 0 ? 4 : dtype == 1 ? 8 : dtype == 2 ? 8 : 16; }

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
    int64_t spanA, spanB, spanC;  // bytes of one problem's operand span
    int elt;
};

struct Candidate {
    bool ok = false;
    double total = 1e300;
    double group = 0;
    int64_t memops = 0;
    int area = 0;
    int P = 0, S = 0, W = 0, ctas = 1;
    int family = IAAT_FAM_FMA;
    DimSplit ms, ns;
    int capA = 0, capB = 0, capC = 0, slotA = 0, slotB = 0, slotC = 0, modeA = 0, modeB = 0, modeC = 0;
    int c_in_smem = 0;
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

// ---------------------------------------------------------------- smem model
// Shared-memory wavefronts of one warp-wide load: lanes request `width`
// bytes at byte offsets addr[l]; 32 banks x 4 B; identical words broadcast.
// Measured on B200 (ncu "L1 Wavefronts Shared"): 128-bit loads are served
// per HALF-warp (each half >= 1 wavefront), narrower loads per warp; inside
// a group, wavefronts = max over banks of the distinct words that bank serves.
int wf_group(const int64_t *addr, int width, int l0, int l1)
{
    int64_t words[32][64];
    int cnt[32] = {0};
    int worst = 1;
    for (int l = l0; l < l1; ++l) {
        for (int w = 0; w < width / 4; ++w) {
            const int64_t word = addr[l] / 4 + w;
            const int b = (int)(word & 31);
            bool seen = false;
            for (int q = 0; q < cnt[b]; ++q)
                if (words[b][q] == word) {
                    seen = true;
                    break;
                }
            if (!seen && cnt[b] < 64) {
                words[b][cnt[b]++] = word;
                worst = std::max(worst, cnt[b]);
            }
        }
    }
    return worst;
}

int wavefronts(const int64_t *addr, int width, int nl)
{
    if (width == 16) return wf_group(addr, width, 0, nl / 2) + wf_group(addr, width, nl / 2, nl);
    return wf_group(addr, width, 0, nl);
}

struct ClassCost {
    double instr = 0;   // warp instructions of one tile pass (whole K + epilogue)
    double wf = 0;      // smem wavefronts of one tile pass
    double single = 0;  // latency-bound duration of one warp's tile pass (cycles)
};

// Lane -> (local problem, tile row, tile col) of the first warp of a class
// under a mapping (see fma_class_loop): map = -2 linear row-fastest, -1 linear
// column-fastest, bm > 0 blocked bm x (32/bm).
struct Lanes {
    int pl[32], ti[32], tj[32];
    int active;
};

Lanes lane_map(int map, int tiles, int tm, int tn)
{
    Lanes L;
    L.active = 0;
    for (int l = 0; l < 32; ++l) {
        if (map < 0) {
            L.pl[l] = l / tiles;
            const int t = l % tiles;
            L.ti[l] = map == -1 ? t / tn : t % tm;
            L.tj[l] = map == -1 ? t % tn : t / tm;
        } else {
            L.pl[l] = 0;
            L.ti[l] = l % map;
            L.tj[l] = l / map;
        }
        const bool ok = L.ti[l] < tm && L.tj[l] < tn;
        if (!ok) {  // idle lane: park it on tile (0,0) (its loads are not issued)
            L.ti[l] = 0;
            L.tj[l] = 0;
        }
        L.active += ok;
    }
    return L;
}

// Warps a class needs for P problems under a mapping.
int class_warps(int map, int P, int tiles, int tm, int tn)
{
    if (map < 0) return (P * tiles + 31) / 32;
    const int bn = 32 / map;
    return P * ((tm + map - 1) / map) * ((tn + bn - 1) / bn);
}

// Cost of one warp of an FMA class: simulate the mapping of the first warp
// and count load instructions and their smem wavefronts for one KU k-block,
// then scale to K.
ClassCost fma_class_cost(const PlanRequest &r, bool vec, int elt, int mr, int nr, const Lanes &L, int row_base,
                         int col_base, int64_t pstrideA, int64_t pstrideB, int64_t pstrideC)
{
    const int VW = 16 / elt, KU = VW;
    const bool TA = r.transA == 1, TB = r.transB == 1;
    int64_t offA[32], offB[32], offC[32];
    int row0[32], col0[32];
    for (int l = 0; l < 32; ++l) {
        row0[l] = row_base + L.ti[l] * mr;
        col0[l] = col_base + L.tj[l] * nr;
        offA[l] = L.pl[l] * pstrideA;
        offB[l] = L.pl[l] * pstrideB;
        offC[l] = L.pl[l] * pstrideC;
    }
    int64_t ad[32];
    double ninstr = 0, nwf = 0;
    // one KU block of op(A): tile-contiguous unless TA
    auto operand = [&](bool kcontig, int R, const int *r0, const int64_t *off, int64_t ld) {
        if (!kcontig) {
            const bool v = vec && R % VW == 0;
            for (int kk = 0; kk < KU; ++kk) {
                const int nld = v ? R / VW : R;
                for (int q = 0; q < nld; ++q) {
                    for (int l = 0; l < 32; ++l)
                        ad[l] = off[l] + (int64_t)(r0[l] + (v ? q * VW : q) + kk * ld) * elt;
                    ninstr += 1;
                    nwf += wavefronts(ad, v ? 16 : elt, 32);
                }
            }
        } else {
            for (int i = 0; i < R; ++i) {
                const int nld = vec ? 1 : KU;
                for (int q = 0; q < nld; ++q) {
                    for (int l = 0; l < 32; ++l) ad[l] = off[l] + (int64_t)(q + (r0[l] + i) * ld) * elt;
                    ninstr += 1;
                    nwf += wavefronts(ad, vec ? 16 : elt, 32);
                }
            }
        }
    };
    operand(TA, mr, row0, offA, r.lda);
    operand(!TB, nr, col0, offB, r.ldb);
    const double nblocks = (double)r.K / KU;
    ClassCost c;
    c.instr = nblocks * (ninstr + (double)KU * mr * nr + 2);
    c.wf = nblocks * nwf;
    // epilogue: C_in smem loads (beta != 0), FMUL/FFMA, global stores
    const bool vc = vec && mr % VW == 0;
    if (!r.beta_zero) {
        double wf = 0;
        for (int j = 0; j < nr; ++j)
            for (int q = 0; q < (vc ? mr / VW : mr); ++q) {
                for (int l = 0; l < 32; ++l)
                    ad[l] = offC[l] + (int64_t)(row0[l] + (vc ? q * VW : q) + (col0[l] + j) * r.ldc) * elt;
                wf += wavefronts(ad, vc ? 16 : elt, 32);
            }
        c.wf += wf;
        c.instr += nr * (vc ? mr / VW : mr);
    }
    c.instr += mr * nr * (r.beta_zero ? 1 : 2) + nr * (vc ? mr / VW : mr) + 60;
    c.single = c.instr + nblocks * 30.0 + 200.0;
    return c;
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

// SM model constants (cycles at ~1.9 GHz), calibrated on B200 sweeps
// (tools/sweep.py; profiles/ round 1).
constexpr double kLoadLatency = 2200.0;   // issue -> full for a bulk-copied stage (besides size/BW)
constexpr double kIssuePerClk = 4.0;      // warp instructions per SM per clock (4 SMSPs)
constexpr double kIssuePerWarp = 0.45;    // sustained issue of one warp (LDS/FMA latency, MIO)
constexpr double kSmemPerClk = 1.0;       // smem wavefronts per SM per clock
constexpr double kGroupFixed = 500.0;     // per-group barrier / dispatch / epilogue tail
constexpr double kGlobalCinPenalty = 1500.0;  // exposed L2/HBM latency of C_in read in the epilogue
constexpr double kOverlapLoss = 0.3;      // fraction of the shorter of (memory, compute) not hidden

struct Knobs {
    int p = 0, s = 0, ctas = 0, mr = 0, nr = 0, fam = -1, order = -1, csmem = -1;
    bool any() const { return p || s || ctas || mr || fam >= 0 || order >= 0 || csmem >= 0; }
};

Plan make_plan_knobs(const PlanRequest &r, const Knobs &kn);
bool plan_ks(const PlanRequest &r, const Knobs &kn, Plan &out);
bool plan_ksg(const PlanRequest &r, const Knobs &kn, Plan &out);
bool plan_ksgs(const PlanRequest &r, const Knobs &kn, Plan &out);

// ---------------------------------------------------------------- install-time tuning table
// tuning/b200.tsv next to libiaat.so (written by paper_2208_09822_b200/tune.py on
// a B200: the install-time stage's "automatically tunes kernels based on
// features of the hardware").  One line per tuned input:
//   dtype tA tB M N K lda ldb ldc packed beta0 vec : mr nr P S ctas order family [csmem]
struct TunedKey {
    int v[12];
    bool operator<(const TunedKey &o) const { return std::lexicographical_compare(v, v + 12, o.v, o.v + 12); }
};

const std::map<TunedKey, Knobs> &tuning_table()
{
    static std::map<TunedKey, Knobs> table;
    static std::once_flag once;
    std::call_once(once, [] {
        std::string path;
        if (const char *e = std::getenv("IAAT_TUNING")) {
            path = e;
        } else {
            Dl_info info;
            if (dladdr((void *)&tuning_table, &info) && info.dli_fname) {
                path = info.dli_fname;
                const size_t slash = path.find_last_of('/');
                path = (slash == std::string::npos ? std::string(".") : path.substr(0, slash)) + "/tuning/b200.tsv";
            }
        }
        FILE *f = path.empty() ? nullptr : std::fopen(path.c_str(), "r");
        if (!f) return;
        char line[512];
        while (std::fgets(line, sizeof line, f)) {
            if (line[0] == '#') continue;
            TunedKey k;
            Knobs kn;
            int n = std::sscanf(line, "%d %d %d %d %d %d %d %d %d %d %d %d : %d %d %d %d %d %d %d %d", &k.v[0],
                                &k.v[1], &k.v[2], &k.v[3], &k.v[4], &k.v[5], &k.v[6], &k.v[7], &k.v[8], &k.v[9],
                                &k.v[10], &k.v[11], &kn.mr, &kn.nr, &kn.p, &kn.s, &kn.ctas, &kn.order, &kn.fam,
                                &kn.csmem);
            if (n == 19) kn.csmem = -1;
            if (n >= 19) table[k] = kn;
        }
        std::fclose(f);
    });
    return table;
}

// ---------------------------------------------------------------- ksg family
// (csrc/iaat_ksg.cuh).  One catalog entry = one kernel: a lane grid
// lr x (32/lr) of mr x nr register tiles, warp blocks of (lr*mr) x
// ((32/lr)*nr) elements of one problem, g groups of w consumer warps.  The
// planner tiles the smallest Mv x Nv >= M x N that the entry's warp blocks
// cover (Mv = M, Nv = N when the lane grid is exact; otherwise the copy
// engine's zero fill supplies the rows / columns past M / N and the TMA
// store clips them), sizes the stage ring to shared memory and picks the
// entry with the lowest modelled time.

// Shared-memory wavefronts of the epilogue's C-buffer accesses of one warp
// for column pitch cp (128-bit accesses run in 4 phases of 8 lanes, 64-bit in
// 2 of 16, 32-bit in 1 of 32; per phase the largest number of distinct words
// in one bank).
int ksg_epi_wavefronts(const IaatKsgCatalogEntry &e, int cp)
{
    const int LR = e.lr, LC = 32 / LR;
    const bool AK = e.trans >= 2, BK = (e.trans & 1) == 0;
    const int VA = AK ? 1 : (e.mr % 4 == 0 ? 4 : (e.mr % 2 == 0 ? 2 : 1));
    const int VB = BK ? 1 : (e.nr % 4 == 0 ? 4 : (e.nr % 2 == 0 ? 2 : 1));
    auto row = [&](int ti) { return AK ? ti : VA * ti; };
    auto col = [&](int tj, int c) { return BK ? tj + LC * c : VB * (tj + LC * (c / VB)) + c % VB; };
    const int V = (!AK && VA >= 2) ? VA : 1;
    const int nph = V == 4 ? 4 : (V == 2 ? 2 : 1), per = 32 / nph;
    int tot = 0;
    for (int c = 0; c < e.nr; ++c)
        for (int ph = 0; ph < nph; ++ph) {
            int words[32][32];
            int nb[32] = {0};
            for (int l = ph * per; l < (ph + 1) * per; ++l) {
                const int w0 = col(l / LR, c) * cp + row(l % LR);
                for (int q = 0; q < V; ++q) {
                    const int w = w0 + q, b = w & 31;
                    bool seen = false;
                    for (int x = 0; x < nb[b]; ++x) seen |= words[b][x] == w;
                    if (!seen && nb[b] < 32) words[b][nb[b]++] = w;
                }
            }
            int mx = 0;
            for (int b = 0; b < 32; ++b) mx = std::max(mx, nb[b]);
            tot += mx;
        }
    return tot;
}

bool ksg_default(const PlanRequest &r)
{
    return r.dtype == 0 && !r.ptr_array && std::min(r.M, r.N) >= 32 && r.K >= 16 &&
           !(r.transA == 1 && r.transB == 0) && !std::getenv("IAAT_NO_KSG");
}

bool ksgs_default(const PlanRequest &r)
{
    return r.dtype == 0 && !r.ptr_array && std::min(r.M, r.N) >= 24 && r.K >= 8 &&
           !(r.transA == 1 && r.transB == 0) && std::getenv("IAAT_KSGS_DEFAULT");
}

bool plan_ksg(const PlanRequest &r, const Knobs &kn, Plan &out)
{
    if (r.ptr_array || r.dtype != 0) return false;
    const int elt = 4;
    const int64_t M = r.M, N = r.N, K = r.K;
    const bool AK = r.transA == 1, BK = r.transB == 0;
    const int64_t colsA = AK ? M : K, colsB = BK ? N : K, rowsA = AK ? K : M, rowsB = BK ? K : N;
    auto al16 = [&](int64_t el) { return (el * elt) % 16 == 0; };
    if (K < 1 || r.batch < 1 || r.batch >= ((int64_t)1 << 31)) return false;
    // TMA boxes for A, B and C: 16-byte aligned bases and strides, no broadcast strides
    if (r.align % 16) return false;
    if (r.batch > 1 && (!al16(r.sA) || !al16(r.sB) || !al16(r.sC) || r.sA < r.lda * colsA ||
                        r.sB < r.ldb * colsB || r.sC < r.ldc * N))
        return false;
    // ... and 16-byte ld's.  The TMA store of C writes whole 16-byte granules
    // along M (measured: rows M .. round_up(M, 4) - 1 of an ld-padded C were
    // overwritten), so C columns must end on a granule boundary.
    bool pv = false;
    if (M % 4 || !al16(r.lda) || !al16(r.ldb) || !al16(r.ldc)) {
        // Column-pair boxes (csrc/iaat_ksg.cuh PV, IaatKsgParams::pairv): even
        // ld's that are not multiples of 4 (n = 2 mod 4) give 8-byte column
        // pitches, which no TMA stride can express -- but TWO columns are a
        // 16-byte multiple.  The operand is described as rows of 2 * ld
        // elements (column pairs).  An MN-major operand (and C) must be packed
        // (ld = rows, so that a pair row holds exactly two columns and the
        // smem pitch stays uniform) with an even column count; a K-major one
        // needs an even ld and an even column count (its dim 0 is ld + K:
        // the odd column of the last pair ends where the problem ends).
        // (a K-major operand with a padded even ld would work the same way; it
        // is left to the slab family until a test covers it)
        auto pair_ok = [&](bool kmaj, int64_t rows, int64_t cols, int64_t ld) {
            if (ld % 2 || cols % 2 || ld != rows) return false;
            return kmaj || 2 * ld <= 256;
        };
        if (std::getenv("IAAT_NO_PAIRV")) return false;
        if (M % 2 || N % 2 || r.ldc != M || 2 * M > 256) return false;
        if (!pair_ok(AK, rowsA, colsA, r.lda) || !pair_ok(BK, rowsB, colsB, r.ldb)) return false;
        pv = true;
    }
    const int64_t lim = (int64_t)1 << 40;
    if (r.sA * elt >= lim || r.sB * elt >= lim || r.sC * elt >= lim) return false;
    const int tidx = r.transA * 2 + r.transB;
    const int nent = (int)(sizeof(kKsgCatalog) / sizeof(kKsgCatalog[0]));
    struct Cand {
        int idx = -1, Mv = 0, Nv = 0, P = 0, S = 0, cp = 0, bm = 0, wpp = 0, stage = 0, cbytes = 0, a_reg = 0, b_reg = 0;
        double cost = 0;
    } best;
    const double bytes = (double)(M * K + K * N + M * N * (r.beta_zero ? 1 : 2)) * elt;
    for (int i = 0; i < nent; ++i) {
        const IaatKsgCatalogEntry &e = kKsgCatalog[i];
        if (e.trans != tidx) continue;
        if (kn.fam == IAAT_FAM_KSG && kn.order >= 0 && kn.order != i) continue;
        if (kn.mr && (e.mr != kn.mr || e.nr != kn.nr)) continue;
        const int LC = 32 / e.lr, BR = e.lr * e.mr, BC = LC * e.nr;
        const int Mv = (int)round_up(M, BR), Nv = (int)round_up(N, BC);
        if (Mv > 256 || Nv > 256) continue;
        const int bm = Mv / BR, wpp = bm * (Nv / BC);
        if (wpp > e.w || e.w % wpp) continue;
        const int P = e.w / wpp;
        int cp = Mv, bestwf = 1 << 30;
        for (int pad = 0; pad < 32 && Mv + pad <= 256 && !pv; pad += 4) {
            const int wf = ksg_epi_wavefronts(e, Mv + pad);
            if (wf < bestwf) bestwf = wf, cp = Mv + pad;
        }
        if (pv) cp = (int)M;  // the C buffer is the packed pair box: columns M apart
        // pv: MN-major boxes hold the packed columns (pitch ld = rows), K-major
        // ones two unswizzled half boxes of Mv / 2 (Nv / 2) rows of kc + 4
        // elements (the odd columns' box starts ld % 4 elements early: TMA box
        // starts are 16-byte aligned)
        const int a_tx = pv ? P * (AK ? Mv * (e.kc + 4) : (int)r.lda * e.kc) * elt : P * Mv * e.kc * elt;
        const int b_tx = pv ? P * (BK ? Nv * (e.kc + 4) : (int)r.ldb * e.kc) * elt : P * Nv * e.kc * elt;
        const int c_tx = P * Nv * cp * elt;
        // (pv boxes are all unswizzled: 128-byte alignment is enough, and the
        // smaller regions buy ring depth -- n = 54: S = 1 -> 2)
        const int ral = pv ? 128 : 1024;
        const int a_reg = (int)(pv && AK ? 2 * round_up(a_tx / 2, ral) : round_up(a_tx, ral));
        const int b_reg = (int)(pv && BK ? 2 * round_up(b_tx / 2, ral) : round_up(b_tx, ral));
        const int stage = a_reg + b_reg, cbytes = (int)round_up(c_tx, ral);
        int S = 0;
        while (S < IAAT_KSG_MAX_STAGES && IAAT_KSG_BAR_BYTES + 1024 + e.g * ((S + 1) * stage + cbytes) <= IAAT_SMEM_LIMIT)
            ++S;
        if (kn.fam == IAAT_FAM_KSG && kn.s > 0) S = std::min(S, kn.s);
        if (S < 1) continue;
        // model: FFMA2 work on the Mv x Nv tile (plain FFMA without a vector
        // operand to pair), against the HBM time of the real bytes; the
        // shorter of the two is partly exposed, and a one-stage ring or a
        // smem-hungry tile (4(mr+nr)/(mr nr) words per FMA) costs extra
        const bool pair = (!AK && e.mr % 2 == 0) || (!BK && e.nr % 2 == 0);
        const double fma = (double)Mv * Nv * K / (128.0 * (pair ? 0.68 : 0.5));
        const double smemf = 4.0 * (e.mr + e.nr) / (e.mr * e.nr);
        const double hbm = bytes / 22.0;
        double t = std::max(fma * std::max(1.0, smemf / 0.9), hbm) + 0.35 * std::min(fma, hbm);
        if (S == 1) t *= 1.2;
        if (best.idx < 0 || t < best.cost) {
            best.idx = i;
            best.Mv = Mv;
            best.Nv = Nv;
            best.P = P;
            best.S = S;
            best.cp = cp;
            best.bm = bm;
            best.wpp = wpp;
            best.stage = stage;
            best.cbytes = cbytes;
            best.a_reg = a_reg;
            best.b_reg = b_reg;
            best.cost = t;
        }
    }
    if (best.idx < 0) return false;
    const IaatKsgCatalogEntry &e = kKsgCatalog[best.idx];
    Plan pl;
    IaatKsgParams &k = pl.kgp;
    k.batch = r.batch;
    k.nunits = (r.batch + best.P - 1) / best.P;
    k.M = (int)M;
    k.N = (int)N;
    k.K = (int)K;
    k.Mv = best.Mv;
    k.Nv = best.Nv;
    k.P = best.P;
    k.S = best.S;
    k.nchunks = (int)((K + e.kc - 1) / e.kc);
    k.a_pitch = pv && !AK ? (int)r.lda : best.Mv;
    k.b_pitch = pv && !BK ? (int)r.ldb : best.Nv;
    k.c_pitch = best.cp;
    k.a_tx = pv && AK ? best.P * best.Mv * (e.kc + 4) * elt : best.P * k.a_pitch * e.kc * elt;
    k.b_tx = pv && BK ? best.P * best.Nv * (e.kc + 4) * elt : best.P * k.b_pitch * e.kc * elt;
    k.a_bytes = best.a_reg;
    k.b_bytes = best.b_reg;
    k.pairv = pv ? 1 : 0;
    k.a_half = pv && AK ? best.a_reg / 2 : 0;
    k.b_half = pv && BK ? best.b_reg / 2 : 0;
    k.lda = (int)r.lda;
    k.ldb = (int)r.ldb;
    k.ldc = (int)r.ldc;
    k.stage_bytes = best.stage;
    k.c_tx = best.P * best.Nv * best.cp * elt;
    k.c_bytes = best.cbytes;
    k.group_bytes = best.S * best.stage + best.cbytes;
    k.beta_zero = r.beta_zero;
    k.bm = best.bm;
    k.wpp = best.wpp;
    auto geo = [&](TmaGeo &g, int64_t rows, int64_t cols, int64_t ld, int64_t stride, bool kmaj, int D) {
        g.dim[0] = (uint64_t)rows;
        g.dim[1] = (uint64_t)cols;
        g.dim[2] = (uint64_t)r.batch;
        g.stride[0] = (uint64_t)(ld * elt);
        g.stride[1] = (uint64_t)((r.batch > 1 ? stride : round_up(ld * cols, 4)) * elt);
        if (kmaj) {
            g.box[0] = (uint32_t)e.kc;
            g.box[1] = (uint32_t)D;
        } else {
            g.box[0] = (uint32_t)D;
            g.box[1] = (uint32_t)e.kc;
        }
        if (pv) {
            // rows of column pairs; a K-major half box takes KC elements of
            // the even (coordinate k0) or odd (ld + k0) columns of D / 2 pairs
            g.dim[0] = (uint64_t)(kmaj ? ld + rows : 2 * ld);
            g.dim[1] = (uint64_t)(cols / 2);
            g.stride[0] = (uint64_t)(2 * ld * elt);
            if (kmaj) {
                g.box[0] = (uint32_t)(e.kc + 4);
                g.box[1] = (uint32_t)(D / 2);
            } else {
                g.box[0] = (uint32_t)(2 * ld);
                g.box[1] = (uint32_t)(e.kc / 2);
            }
        }
        g.box[2] = (uint32_t)best.P;
        g.swizzle128 = kmaj && e.kc == 32 && !pv ? 1 : 0;
        g.swizzle64 = kmaj && e.kc == 16 && !pv ? 1 : 0;
    };
    geo(pl.tmA, rowsA, colsA, r.lda, r.sA, AK, best.Mv);
    geo(pl.tmB, rowsB, colsB, r.ldb, r.sB, BK, best.Nv);
    pl.tmC.dim[0] = (uint64_t)M;
    pl.tmC.dim[1] = (uint64_t)N;
    pl.tmC.dim[2] = (uint64_t)r.batch;
    pl.tmC.stride[0] = (uint64_t)(r.ldc * elt);
    pl.tmC.stride[1] = (uint64_t)((r.batch > 1 ? r.sC : round_up(r.ldc * N, 4)) * elt);
    pl.tmC.box[0] = (uint32_t)best.cp;
    pl.tmC.box[1] = (uint32_t)best.Nv;
    pl.tmC.box[2] = (uint32_t)best.P;
    if (pv) {
        pl.tmC.dim[0] = (uint64_t)(2 * M);
        pl.tmC.dim[1] = (uint64_t)(N / 2);
        pl.tmC.stride[0] = (uint64_t)(2 * M * elt);
        pl.tmC.box[0] = (uint32_t)(2 * M);
        pl.tmC.box[1] = (uint32_t)(best.Nv / 2);
    }
    pl.ksg = 1;
    pl.kg_entry = best.idx;
    pl.family = IAAT_FAM_KSG;
    pl.vec = 1;
    pl.ctas = 1;
    pl.grid = (int)std::min<int64_t>((k.nunits + e.g - 1) / e.g, (int64_t)r.sm_count);
    pl.block = 128 + 32 * e.g * e.w;  // IAAT_KSG_THREADS_OF(g * w): producer warpgroup + consumers
    pl.smem = IAAT_KSG_BAR_BYTES + 1024 + e.g * k.group_bytes;
    pl.est_total = best.cost;
    // the paper's cost over the Mv x Nv tiling: smem words
    // the lanes' tiles read per k-step, plus the C traffic
    pl.memops = (int64_t)(best.Mv / e.mr) * (best.Nv / e.nr) * (e.mr + e.nr) * K + 2 * M * N;
    pl.status = 0;
    out = pl;
    return true;
}


// ksgs (slab-staged lane grids, csrc/iaat_ksg.cuh): inputs the TMA rules
// exclude.  A unit's P packed problems are one stage (one bulk copy per
// operand of the enclosing 16-byte-aligned span, whole K); tiles cover
// Mv x Nv >= M x N and the stage keeps enough slack after the span for the
// padded rows / columns to read (never stored).
bool plan_ksgs(const PlanRequest &r, const Knobs &kn, Plan &out)
{
    if (r.ptr_array || r.dtype != 0) return false;
    const int elt = 4;
    const int64_t M = r.M, N = r.N, K = r.K;
    const bool AK = r.transA == 1, BK = r.transB == 0;
    const int64_t colsA = AK ? M : K, colsB = BK ? N : K, rowsA = AK ? K : M, rowsB = BK ? K : N;
    if (K < 1 || r.batch < 1 || r.batch >= ((int64_t)1 << 31)) return false;
    // packed (or nearly): the unit's span is the problems' bytes
    if (r.batch > 1 && (r.sA < r.lda * colsA || r.sB < r.ldb * colsB || r.sC < r.ldc * N ||
                        r.sA > r.lda * colsA + 16 || r.sB > r.ldb * colsB + 16))
        return false;
    const int tidx = r.transA * 2 + r.transB;
    const int nent = (int)(sizeof(kKsgsCatalog) / sizeof(kKsgsCatalog[0]));
    struct Cand {
        int idx = -1, Mv = 0, Nv = 0, P = 0, S = 0, bm = 0, wpp = 0, ab = 0, bb = 0, cb = 0;
        double cost = 0;
    } best;
    const double bytes = (double)(M * K + K * N + M * N * (r.beta_zero ? 1 : 2)) * elt;
    const int64_t sA = r.batch > 1 ? r.sA : r.lda * colsA, sB = r.batch > 1 ? r.sB : r.ldb * colsB;
    // C through the stage (C_in bulk-loaded with A and B, C bulk-stored by the
    // producer): only where a unit's C is one gap-free span (ldc == M, packed
    // problems), so that the span store writes nothing but C elements
    const bool cpack = r.ldc == M && (r.batch <= 1 || r.sC == M * N);
    const bool csm = cpack && !(kn.fam == IAAT_FAM_KSGS && kn.csmem == 0);
    for (int i = 0; i < nent; ++i) {
        const IaatKsgsCatalogEntry &e = kKsgsCatalog[i];
        if (e.trans != tidx) continue;
        if (kn.fam == IAAT_FAM_KSGS && kn.order >= 0 && kn.order != i) continue;
        const int LC = 32 / e.lr, BR = e.lr * e.mr, BC = LC * e.nr;
        const int Mv = (int)round_up(M, BR), Nv = (int)round_up(N, BC);
        const int bm = Mv / BR, wpp = bm * (Nv / BC);
        if (wpp > e.w || e.w % wpp) continue;
        const int P = e.w / wpp;
        // span of P problems + the 16-byte realignment + the padded reads' slack
        const int64_t spanA = ((int64_t)(P - 1) * sA + (colsA - 1) * r.lda + rowsA) * elt;
        const int64_t spanB = ((int64_t)(P - 1) * sB + (colsB - 1) * r.ldb + rowsB) * elt;
        const int64_t slackA = (AK ? (int64_t)(Mv - M) * r.lda : (Mv - M)) * elt;
        const int64_t slackB = (BK ? (int64_t)(Nv - N) * r.ldb : (Nv - N)) * elt;
        const int ab = (int)round_up(spanA + 32 + slackA, 128), bb = (int)round_up(spanB + 32 + slackB, 128);
        // (no CS instance for 10 x 10 tiles: gen/generate.py ksgs_cs)
        const int cb = csm && e.mr * e.nr < 100 ? (int)round_up((int64_t)P * M * N * elt + 32, 128) : 0;
        const int stage = ab + bb + cb;
        // one ring of S stages shared by the e.g groups (csrc/iaat_ksg.cuh SmemS)
        int S = 0;
        while (S < IAAT_KSGS_MAX_STAGES && IAAT_KSG_BAR_BYTES + 1024 + (S + 1) * stage <= IAAT_SMEM_LIMIT) ++S;
        if (kn.fam == IAAT_FAM_KSGS && kn.s > 0) S = std::min(S, kn.s);
        if (S < 1) continue;
        // units in flight beyond the G being computed: the loads they hide
        const int ahead = S - e.g;
        // scalar loads: (mr + nr) LDS per k-step beside mr*nr/2 FFMA2
        const bool pair = e.mr % 2 == 0 || e.nr % 2 == 0;  // odd x odd: all but one row / column paired
        const double fma = (double)P * Mv * Nv * K / (128.0 * (pair ? 0.6 : 0.55)) / P;
        const double smemf = 4.0 * (e.mr + e.nr) / (e.mr * e.nr);
        const double hbm = bytes / 22.0;
        double t = std::max(fma * std::max(1.0, smemf / 0.9), hbm) + 0.35 * std::min(fma, hbm);
        if (ahead < 1) t *= 1.6;
        else if (ahead < 2) t *= 1.15;
        if (best.idx < 0 || t < best.cost) {
            best.idx = i;
            best.Mv = Mv;
            best.Nv = Nv;
            best.P = P;
            best.S = S;
            best.bm = bm;
            best.wpp = wpp;
            best.ab = ab;
            best.bb = bb;
            best.cb = cb;
            best.cost = t;
        }
    }
    if (best.idx < 0) return false;
    const IaatKsgsCatalogEntry &e = kKsgsCatalog[best.idx];
    Plan pl;
    IaatKsgParams &k = pl.kgp;
    k.batch = r.batch;
    k.nunits = (r.batch + best.P - 1) / best.P;
    k.M = (int)M;
    k.N = (int)N;
    k.K = (int)K;
    k.Mv = best.Mv;
    k.Nv = best.Nv;
    k.P = best.P;
    k.S = best.S;
    k.nchunks = 1;
    k.a_bytes = best.ab;
    k.b_bytes = best.bb;
    k.stage_bytes = best.ab + best.bb + best.cb;
    k.c_bytes = best.cb;  // 0: C through global
    k.group_bytes = best.S * k.stage_bytes;
    k.beta_zero = r.beta_zero;
    k.bm = best.bm;
    k.wpp = best.wpp;
    k.sA = sA;
    k.sB = sB;
    k.sC = r.batch > 1 ? r.sC : r.ldc * N;
    k.lda = (int)r.lda;
    k.ldb = (int)r.ldb;
    k.ldc = (int)r.ldc;
    pl.ksg = 2;
    pl.kg_entry = best.idx;
    pl.family = IAAT_FAM_KSGS;
    pl.vec = 0;
    pl.ctas = 1;
    pl.grid = (int)std::min<int64_t>((k.nunits + e.g - 1) / e.g, (int64_t)r.sm_count);
    pl.block = 128 + 32 * e.g * e.w;
    pl.smem = IAAT_KSG_BAR_BYTES + 1024 + k.group_bytes;
    pl.est_total = best.cost;
    pl.memops = (int64_t)(best.Mv / e.mr) * (best.Nv / e.nr) * (e.mr + e.nr) * K + 2 * M * N;
    pl.status = 0;
    out = pl;
    return true;
}

Plan make_plan(const PlanRequest &r)
{
    Knobs kn;
    // Test/tuning knobs (never needed in production): force P, S, CTAs/SM,
    // the first strip sizes, the lane mapping or the family, e.g.
    // IAAT_FORCE_P=4 IAAT_FORCE_TILE=8x8.
    auto envi = [](const char *n) { const char *v = std::getenv(n); return v ? std::atoi(v) : 0; };
    kn.p = envi("IAAT_FORCE_P");
    kn.s = envi("IAAT_FORCE_S");
    kn.ctas = envi("IAAT_FORCE_CTAS");
    if (const char *ft = std::getenv("IAAT_FORCE_TILE")) std::sscanf(ft, "%dx%d", &kn.mr, &kn.nr);
    kn.fam = std::getenv("IAAT_FORCE_FAMILY") ? envi("IAAT_FORCE_FAMILY") : -1;
    kn.order = std::getenv("IAAT_FORCE_ORDER") ? envi("IAAT_FORCE_ORDER") : -1;
    kn.csmem = std::getenv("IAAT_FORCE_CSMEM") ? envi("IAAT_FORCE_CSMEM") : -1;
    bool tuned = false;
    if (!kn.any() && !r.ptr_array && !std::getenv("IAAT_NO_TUNING")) {
        const int elt = elt_of(r.dtype);
        const int64_t colsA = r.transA ? r.M : r.K, colsB = r.transB ? r.K : r.N;
        const bool packed = r.batch <= 1 || (r.sA == r.lda * colsA && r.sB == r.ldb * colsB && r.sC == r.ldc * r.N);
        auto al16 = [&](int64_t el) { return (el * elt) % 16 == 0; };
        const bool vec = r.align % 16 == 0 && al16(r.lda) && al16(r.ldb) && al16(r.ldc) &&
                         (r.batch <= 1 || (al16(r.sA) && al16(r.sB) && al16(r.sC)));
        TunedKey k{{r.dtype, r.transA, r.transB, (int)r.M, (int)r.N, (int)r.K, (int)r.lda, (int)r.ldb, (int)r.ldc,
                    packed ? 1 : 0, r.beta_zero, vec ? 1 : 0}};
        const auto &t = tuning_table();
        auto it = t.find(k);
        if (it != t.end()) {
            kn = it->second;
            tuned = true;
        }
    }
    if (!kn.any() && (r.dtype == 1 || r.dtype == 3) && r.M % 8 == 0 && r.N % 8 == 0) {
        // fp64 on tensor cores: the K-streamed DMMA family is the default
        // wherever its TMA preconditions hold (measured 1.3-2.5x the slab
        // DMMA kernels on B200, profiles/)
        Knobs kd;
        kd.fam = IAAT_FAM_KS_DMMA;
        Plan pd;
        if (plan_ks(r, kd, pd)) return pd;
    }
    if (kn.fam == IAAT_FAM_KSG) {
        Plan pg;
        if (plan_ksg(r, kn, pg)) {
            pg.tuned = tuned;
            return pg;
        }
        kn = Knobs();
    }
    if (kn.fam == IAAT_FAM_KSGS) {
        Plan pg;
        if (plan_ksgs(r, kn, pg)) {
            pg.tuned = tuned;
            return pg;
        }
        kn = Knobs();
    }
    if (!kn.any() && ksg_default(r)) {
        // the upper half of the fp32 domain: lane-grid register tiles with
        // warp groups (csrc/iaat_ksg.cuh) wherever their TMA rules hold.
        // (The slab-staged ksgs kernels are chosen only by the install-time
        // table: on held-out misaligned shapes they measured no better than
        // the slab family on average, profiles/r02/heldout_r02*.)
        Plan pg;
        if (plan_ksg(r, Knobs(), pg)) return pg;
    }
    if (!kn.any() && ksgs_default(r)) {
        // the same upper half where the TMA rules fail (odd ld's, misaligned
        // bases): the slab-staged lane grids
        Plan pg;
        if (plan_ksgs(r, Knobs(), pg)) return pg;
    }
    Plan p = make_plan_knobs(r, kn);
    if (p.status != 0 && kn.any()) p = make_plan_knobs(r, Knobs());
    else p.tuned = tuned;
    if (p.status != 0 && !kn.any()) {
        // shapes the slab family cannot stage (e.g. 16 x 16 x 2000: one
        // problem's span exceeds shared memory) stream through the
        // K-streamed families instead
        Knobs kk;
        kk.fam = (r.dtype == 1 || r.dtype == 3) ? IAAT_FAM_KS_DMMA : IAAT_FAM_KS_FMA;
        Plan pk;
        if (plan_ks(r, kk, pk)) return pk;
        if (kk.fam == IAAT_FAM_KS_DMMA) {
            kk.fam = IAAT_FAM_KS_FMA;
            if (plan_ks(r, kk, pk)) return pk;
        }
    }
    return p;
}

Plan make_plan_knobs(const PlanRequest &r, const Knobs &kn)
{
    if (kn.fam == IAAT_FAM_KS_FMA || kn.fam == IAAT_FAM_KS_DMMA || kn.fam == IAAT_FAM_KSU_FMA) {
        Plan ksplan;
        if (plan_ks(r, kn, ksplan)) return ksplan;
        ksplan.status = 5;
        return ksplan;
    }
    Plan plan;
    const int elt = elt_of(r.dtype);
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
    geo.spanC = ((N - 1) * r.ldc + M) * elt;

    // 16-byte vector paths are legal iff every problem's A, B, C base and
    // every column start is 16 B aligned (strided API only).
    auto al16 = [&](int64_t el) { return (el * elt) % 16 == 0; };
    const bool vec = !r.ptr_array && r.align % 16 == 0 && al16(r.lda) && al16(r.ldb) && al16(r.ldc) &&
                     (r.batch <= 1 || (al16(r.sA) && al16(r.sB) && al16(r.sC)));
    plan.vec = vec ? 1 : 0;

    const double hbm_per_problem = (double)(M * K + K * N + M * N * (r.beta_zero ? 1 : 2)) * elt;
    const int64_t sAb = r.sA * elt, sBb = r.sB * elt, sCb = r.sC * elt;

    const int force_s = kn.s, force_c = kn.ctas, force_mr = kn.mr, force_nr = kn.nr;
    const int force_fam = kn.fam, force_order = kn.order;

    Candidate best;
    const int64_t pmax_batch = std::max<int64_t>(1, (r.batch + r.sm_count - 1) / r.sm_count);
    const int force_p = kn.p > 0 ? (int)std::min<int64_t>(kn.p, pmax_batch) : 0;

    // Evaluate one (tiling, P, CTAs/SM) point.  `warp_instr`, `warp_wf`,
    // `single`: per-group totals of the compute warps (see ClassCost).
    auto evaluate = [&](Candidate &c, int P, int ctas, double warp_instr, double warp_wf, double single,
                        double pipe) -> bool {
        const int smem_cta = (int)std::min<int64_t>(IAAT_SMEM_LIMIT, 228 * 1024 / ctas - 1024) - IAAT_BAR_BYTES;
        stage_layout(geo.spanA, sAb, P, r.ptr_array, c.modeA, c.slotA, c.capA);
        stage_layout(geo.spanB, sBb, P, r.ptr_array, c.modeB, c.slotB, c.capB);
        c.capC = 0;
        c.c_in_smem = 0;
        if (!r.beta_zero && kn.csmem != 0) {  // C_in rides in the stage with A and B (read from smem)
            stage_layout(geo.spanC, sCb, P, r.ptr_array, c.modeC, c.slotC, c.capC);
            c.c_in_smem = 1;
        }
        int64_t stage = (int64_t)c.capA + c.capB + c.capC;
        int S = (int)std::min<int64_t>(4, smem_cta / stage);
        if (c.c_in_smem && (S < 1 || (S < 2 && P > 1))) {
            c.capC = 0;  // C_in does not fit: L2-prefetched C_in read from global
            c.c_in_smem = 0;
            stage = (int64_t)c.capA + c.capB;
            S = (int)std::min<int64_t>(4, smem_cta / stage);
        }
        if (force_s > 0) S = (int)std::min<int64_t>(force_s, smem_cta / stage);
        if (S < 1 || (S < 2 && P > 1)) return false;
        c.S = S;
        c.P = P;
        c.ctas = ctas;
        // one "round" = every resident CTA of the SM processes one group
        const double bytes = ctas * P * hbm_per_problem;
        const double t_hbm = bytes / kHbmBytesPerClk;
        const double rate = std::min(kIssuePerClk, kIssuePerWarp * ctas * c.W);
        const double t_issue = ctas * warp_instr / rate;
        const double t_smem = ctas * warp_wf / kSmemPerClk;
        const double t_pipe = ctas * pipe;
        // a stage is refilled only after its group is consumed: S-1 stages
        // must cover the load latency of a stage of this size
        const double t_load = (kLoadLatency + ctas * stage / kHbmBytesPerClk) / (S > 1 ? S - 1 : 1);
        // compute and staging overlap only partly (the whole CTA moves from
        // group to group together): T = max(...) + 0.3 * the overlapped part
        const double t_comp = std::max(std::max(t_issue, t_smem), std::max(t_pipe, single));
        const double t_mem = std::max(t_hbm, t_load);
        double t = std::max(t_mem, t_comp) + kOverlapLoss * std::min(t_hbm, t_comp) + kGroupFixed;
        if (S == 1) t = t_hbm + t_comp + kGroupFixed + kLoadLatency;
        if (!r.beta_zero && !c.c_in_smem) t += kGlobalCinPenalty;  // C_in latency in the epilogue
        const int64_t ngroups = (r.batch + P - 1) / P;
        const int64_t slots = (int64_t)r.sm_count * ctas;
        const int64_t waves = (ngroups + slots - 1) / slots;
        c.group = t;
        c.total = t * (double)waves + 3000.0;  // launch + pipeline fill/drain
        c.ok = true;
        return true;
    };

    // ------------------------------------------------------------ FMA family
    const int maxt = 8;
    auto msplits = splits((int)M, maxt, vw);
    auto nsplits = splits((int)N, maxt, vw);
    const int64_t pstrideA = r.ptr_array ? 0 : sAb, pstrideB = r.ptr_array ? 0 : sBb;
    const int64_t pstrideC = r.ptr_array ? 0 : sCb;
    for (const auto &ms : msplits) {
        for (const auto &ns : nsplits) {
            if (force_fam >= 0 && force_fam != IAAT_FAM_FMA) continue;
            if (force_mr && (ms.s[0].size != force_mr || ns.s[0].size != force_nr)) continue;
            bool avail = true;
            int64_t memops = 2 * M * N;
            int area = 0;
            // mapping options per class: linear row-/column-fastest, blocked bm x 32/bm
            static const int kMaps[8] = {-2, -1, 1, 2, 4, 8, 16, 32};
            struct C4 {
                int mr, nr, tiles, tm, tn, rb, cb;
                ClassCost cost[8];
                bool ok[8];
            } cl[4];
            int ncl = 0;
            int rb = 0;
            for (int a = 0; a < ms.n && avail; ++a) {
                int cb = 0;
                for (int b = 0; b < ns.n; ++b) {
                    const int mr = ms.s[a].size, nr = ns.s[b].size;
                    if (!catalog_has(r.dtype, tidx, IAAT_FAM_FMA, mr, nr)) {
                        avail = false;
                        break;
                    }
                    const int tm = ms.s[a].count, tn = ns.s[b].count;
                    C4 &q = cl[ncl++];
                    q.mr = mr;
                    q.nr = nr;
                    q.tiles = tm * tn;
                    q.tm = tm;
                    q.tn = tn;
                    q.rb = rb;
                    q.cb = cb;
                    for (int m = 0; m < 8; ++m) {
                        const int map = kMaps[m];
                        q.ok[m] = true;
                        if (force_order >= 0 && !((force_order == 0 && map == -2) || (force_order == 1 && map == -1) ||
                                                  (force_order >= 2 && map == force_order - 1)))
                            q.ok[m] = false;
                        // a blocked warp must stay inside one problem and be mostly busy
                        if (map > 0) {
                            Lanes L = lane_map(map, q.tiles, tm, tn);
                            if (L.active < 24 || q.tiles < 32) q.ok[m] = false;
                        }
                        if (!q.ok[m]) continue;
                        Lanes L = lane_map(map, q.tiles, tm, tn);
                        q.cost[m] = fma_class_cost(r, vec, elt, mr, nr, L, rb, cb, pstrideA, pstrideB, pstrideC);
                    }
                    memops += (int64_t)tm * tn * (mr + nr) * K;
                    area = std::max(area, mr * nr);
                    cb += ns.s[b].size * ns.s[b].count;
                }
                rb += ms.s[a].size * ms.s[a].count;
            }
            if (!avail) continue;
            for (int ctas = 1; ctas <= 4; ++ctas) {
                if (force_c && ctas != force_c) continue;
                const int wmax = IAAT_MAX_THREADS / 32 / ctas - 1;
                for (int P = 1; P <= 1024; ++P) {
                    if (P > pmax_batch && P > 1) break;
                    if (force_p && P != force_p) continue;
                    int W = 0;
                    double instr = 0, wf = 0, single = 0;
                    int pick[4];
                    bool fits = true;
                    for (int q = 0; q < ncl; ++q) {
                        // cheapest mapping of this class at this P
                        double bestk = 1e300;
                        pick[q] = -1;
                        for (int m = 0; m < 8; ++m) {
                            if (!cl[q].ok[m]) continue;
                            const int w = class_warps(kMaps[m], P, cl[q].tiles, cl[q].tm, cl[q].tn);
                            const double k =
                                w * std::max(cl[q].cost[m].instr / kIssuePerClk, cl[q].cost[m].wf / kSmemPerClk);
                            if (k < bestk * 0.999) {
                                bestk = k;
                                pick[q] = m;
                            }
                        }
                        if (pick[q] < 0) {
                            fits = false;
                            break;
                        }
                        const int w = class_warps(kMaps[pick[q]], P, cl[q].tiles, cl[q].tm, cl[q].tn);
                        W += w;
                        instr += w * cl[q].cost[pick[q]].instr;
                        wf += w * cl[q].cost[pick[q]].wf;
                        single = std::max(single, cl[q].cost[pick[q]].single);
                    }
                    if (!fits) continue;
                    if (W > wmax) break;
                    double pipe = 0;
                    if (r.dtype == 1) pipe = (double)P * M * N * K / kDfmaPerClk;
                    if (r.dtype == 3) pipe = 4.0 * P * M * N * K / kDfmaPerClk;  // 4 DFMA per complex MAC
                    Candidate c;
                    c.family = IAAT_FAM_FMA;
                    c.ms = ms;
                    c.ns = ns;
                    c.memops = memops;
                    c.area = area;
                    c.W = W;
                    if (!evaluate(c, P, ctas, instr, wf, single, pipe)) continue;
                    if (!better(c, best)) continue;
                    int wb = 0;
                    c.ncls = ncl;
                    for (int q = 0; q < ncl; ++q) {
                        const int map = kMaps[pick[q]];
                        const int w = class_warps(map, P, cl[q].tiles, cl[q].tm, cl[q].tn);
                        c.cls[q] = IaatClass{catalog_code(IAAT_FAM_FMA, cl[q].mr, cl[q].nr), wb, wb + w,
                                             cl[q].tiles, cl[q].tm, cl[q].rb, cl[q].mr, cl[q].cb, cl[q].nr,
                                             cl[q].tn, map == -1 ? 1 : 0, map > 0 ? map : 0};
                        wb += w;
                    }
                    best = c;
                }
            }
        }
    }

    // ------------------------------------------------------------ DMMA family (fp64)
    if (r.dtype == 1 && M % 8 == 0 && N % 8 == 0 && !(force_fam >= 0 && force_fam != IAAT_FAM_DMMA)) {
        for (int wm = 1; wm <= 4; wm *= 2)
            for (int wn = 1; wn <= 4; wn *= 2) {
                if ((M / 8) % wm || (N / 8) % wn) continue;
                if (force_mr && (8 * wm != force_mr || 8 * wn != force_nr)) continue;
                if (!catalog_has(1, tidx, IAAT_FAM_DMMA, 8 * wm, 8 * wn)) continue;
                const int tm = (int)(M / (8 * wm)), tn = (int)(N / (8 * wn));
                const int tiles = tm * tn;
                const int64_t memops = (int64_t)tiles * (8 * wm + 8 * wn) * K + 2 * M * N;
                // per item (one warp tile over K): DMMAs + fragment loads + epilogue
                // per 8 k: 2 WM WN DMMAs, one LDS.128 per k-contiguous fragment
                // (two LDS.64 otherwise), ~6 wavefronts per fragment pair
                const double kst = (double)((K + 7) / 8);
                const double nla = r.transA ? 1.0 : 2.0, nlb = r.transB ? 2.0 : 1.0;
                const double instr_item =
                    kst * (2 * wm * wn + wm * nla + wn * nlb + 4) + wm * wn * (r.beta_zero ? 6 : 10) + 30;
                const double wf_item = kst * (wm + wn) * 6.0 + wm * wn * (r.beta_zero ? 0 : 2);
                for (int ctas = 1; ctas <= 4; ++ctas) {
                    if (force_c && ctas != force_c) continue;
                    const int wmax = IAAT_MAX_THREADS / 32 / ctas - 1;
                    for (int P = 1; P <= 64; ++P) {
                        if (P > pmax_batch && P > 1) break;
                        if (force_p && P != force_p) continue;
                        const int items = P * tiles;
                        for (int W = 2; W <= wmax; ++W) {
                            if (W > items && W > 2) break;
                            const double per_warp = std::ceil((double)items / W);
                            // DMMA pipe: 128 flop / clk / SM at the fp64 peak
                            const double pipe = (double)P * 2.0 * M * N * K / 128.0 * (per_warp * W / items);
                            Candidate c;
                            c.family = IAAT_FAM_DMMA;
                            c.ms.s[0] = {8 * wm, tm};
                            c.ms.n = 1;
                            c.ns.s[0] = {8 * wn, tn};
                            c.ns.n = 1;
                            c.memops = memops;
                            c.area = 64 * wm * wn;
                            c.W = W;
                            const double single = per_warp * (instr_item + kst * 40.0) + 400.0;
                            if (!evaluate(c, P, ctas, per_warp * W * instr_item, per_warp * W * wf_item, single,
                                          pipe))
                                continue;
                            if (!better(c, best)) continue;
                            c.ncls = 1;
                            c.cls[0] = IaatClass{catalog_code(IAAT_FAM_DMMA, 8 * wm, 8 * wn), 0, W, tiles, tm,
                                                 0, 8 * wm, 0, 8 * wn, tn, 0, 0};
                            best = c;
                        }
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
    kp.modeC = best.modeC;
    kp.spanA = (int)geo.spanA;
    kp.spanB = (int)geo.spanB;
    kp.spanC = (int)geo.spanC;
    kp.slotA = best.slotA;
    kp.slotB = best.slotB;
    kp.slotC = best.slotC;
    kp.capA = best.capA;
    kp.capB = best.capB;
    kp.capC = best.capC;
    kp.stage_bytes = best.capA + best.capB + best.capC;
    kp.beta_zero = r.beta_zero;
    kp.c_in_smem = best.c_in_smem;
    kp.prefetch_c = (!r.beta_zero && !best.c_in_smem) ? 1 : 0;
    kp.nclasses = best.ncls;
    for (int q = 0; q < best.ncls; ++q) kp.cls[q] = best.cls[q];
    plan.family = best.family;
    plan.ctas = best.ctas;
    plan.grid = (int)std::min<int64_t>(kp.ngroups, (int64_t)r.sm_count * best.ctas);
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

// ---------------------------------------------------------------- K-streamed family (iaat_ks.cuh)
// Applicability: strided API; every base, ld and problem stride 16 B aligned
// (TMA global-address rules); problems do not overlap; M, N <= 256 (box
// extents).  Units of P problems stream through an S-stage ring of K-chunks
// (kc = 128 B / elt); the same exact strip decomposition as the FMA family
// gives the tile classes.
namespace {

struct KsCand {
    bool ok = false;
    int single = 0;
    int dmma = 0;  // 1: fp64 DMMA warp tiles (one class, one warp tile per warp)
    double total = 1e300, unit = 0;
    int P = 0, S = 0, W = 0, ctas = 1, a_bytes = 0, b_bytes = 0, a_pitch = 0, b_pitch = 0;
    DimSplit ms, ns;
    IaatClass cls[IAAT_MAX_CLASSES];
    int ncls = 0;
    int64_t memops = 0;
};

// smem wavefronts + instructions of one k-block (KU k-steps) of one warp of
// a KS FMA class under lane mapping `map` (see lane_map).
void ks_class_cost(const PlanRequest &r, int elt, int mr, int nr, const Lanes &L, int rb, int cb, int tm, int tn,
                   int a_pitch, int b_pitch, int kc, double &instr, double &wf)
{
    const int VW = 16 / elt, KU = VW;
    const bool AK = r.transA == 1, BK = r.transB == 0;
    int64_t ad[32];
    instr = (double)KU * mr * nr + 4;
    wf = 0;
    auto operand = [&](bool kmaj, int R, bool is_a) {
        const int D = is_a ? (int)r.M : (int)r.N;
        const int pitch = is_a ? a_pitch : b_pitch;
        const int t_n = is_a ? tm : tn;
        const int base = is_a ? rb : cb;
        if (kmaj) {
            for (int i = 0; i < R; ++i) {
                for (int l = 0; l < 32; ++l) {
                    const int t = is_a ? L.ti[l] : L.tj[l];
                    const int64_t rab = (int64_t)L.pl[l] * D + base + t + t_n * i;
                    ad[l] = rab * 128 + (((rab & 7)) << 4);
                }
                wf += wavefronts(ad, 16, 32);
                instr += 2;  // LDS + XOR
            }
        } else {
            const bool v = R % VW == 0;
            for (int kk = 0; kk < KU; ++kk)
                for (int q = 0; q < (v ? R / VW : R); ++q) {
                    for (int l = 0; l < 32; ++l) {
                        const int t = is_a ? L.ti[l] : L.tj[l];
                        ad[l] = ((int64_t)L.pl[l] * kc * pitch + (int64_t)kk * pitch + base + t * R +
                                 (v ? q * VW : q)) * elt;
                    }
                    wf += wavefronts(ad, v ? 16 : elt, 32);
                    instr += 1;
                }
            instr += KU;  // row address adds
        }
    };
    operand(AK, mr, true);
    operand(BK, nr, false);
}

}  // namespace

// ---------------------------------------------------------------- complex fp64 on DMMA (ZGEMM)
// K-streamed TMA boxes over the real view of the interleaved data (an R x C
// complex matrix = a 2R x C real one, ld doubled), kc = 8 complex k-steps per
// chunk: K-major rows of 8 complex = 128 bytes (swizzled), MN-major rows of
// pitch >= 2D doubles with pitch = 8 (mod 16).  One warp tile per warp.
bool plan_ks_zdmma(const PlanRequest &r, const Knobs &kn, Plan &out)
{
    if (!(kn.fam == IAAT_FAM_KS_DMMA || !kn.any())) return false;
    const int64_t M = r.M, N = r.N, K = r.K;
    if (M % 8 || N % 8 || K < 1 || M > 120 || N > 120) return false;
    const bool AK = r.transA == 1, BK = r.transB == 0;
    const int tidx = r.transA * 2 + r.transB;
    const int64_t colsA = AK ? M : K, colsB = BK ? N : K, rowsA = AK ? K : M, rowsB = BK ? K : N;
    if (r.align % 16 != 0) return false;
    if (r.batch > 1 && (r.sA < r.lda * colsA || r.sB < r.ldb * colsB)) return false;
    if (r.batch >= ((int64_t)1 << 31) || r.sA * 16 >= (int64_t)1 << 40 || r.sB * 16 >= (int64_t)1 << 40) return false;
    const int kc = 8, nchunks = (int)((K + kc - 1) / kc);
    auto zpitch = [](int64_t D) { int64_t q = 2 * D; while (q % 16 != 8) ++q; return (int)q; };
    const int da = AK ? 16 : zpitch(M), db = BK ? 16 : zpitch(N);
    const double hbm_per_problem = (double)(M * K + K * N + M * N * (r.beta_zero ? 1 : 2)) * 16;
    KsCand best;
    for (int wm = 1; wm <= 7; ++wm)  // the catalog decides which (wm, wn) exist
        for (int wn = 1; wn <= 7; ++wn) {
            if ((M / 8) % wm || (N / 8) % wn) continue;
            if (kn.mr && (8 * wm != kn.mr || 8 * wn != kn.nr)) continue;
            if (!catalog_has(3, tidx, IAAT_FAM_KS_DMMA, 8 * wm, 8 * wn)) continue;
            const int tm = (int)(M / (8 * wm)), tn = (int)(N / (8 * wn)), tiles = tm * tn;
            for (int ctas = 1; ctas <= 3; ++ctas) {
                if (kn.ctas && ctas != kn.ctas) continue;
                const int wmax = std::min(IAAT_KSD_THREADS(wm, wn) / 32, 16 / ctas) - 1;
                const int smem_cta = (int)std::min<int64_t>(IAAT_SMEM_LIMIT, 228 * 1024 / ctas - 1024);
                for (int P = 1; P * tiles <= wmax; ++P) {
                    if (kn.p && P != kn.p) continue;
                    if (P > 1 && (int64_t)(P - 1) * r.sm_count * ctas >= r.batch) break;
                    const int W = P * tiles;
                    const int a_bytes = (int)round_up((int64_t)P * (AK ? M * 128 : (int64_t)kc * da * 8), 1024);
                    const int b_bytes = (int)round_up((int64_t)P * (BK ? N * 128 : (int64_t)kc * db * 8), 1024);
                    int S = std::min(IAAT_KS_MAX_STAGES, (smem_cta - IAAT_KS_BAR_BYTES - 1024) / (a_bytes + b_bytes));
                    if (kn.s > 0) S = std::min(S, kn.s);
                    if (S < 2) continue;
                    const double t_hbm = ctas * P * hbm_per_problem / kHbmBytesPerClk;
                    const double t_dmma = ctas * 4.0 * P * M * N * K / kDfmaPerClk;  // 4 real products
                    const double t_lat = kLoadLatency * nchunks / std::max(1, S - 1) / ctas;
                    const double t = std::max(std::max(t_hbm, t_dmma), t_lat) + 0.15 * std::min(t_hbm, t_dmma) + 300.0;
                    const int64_t nunits = (r.batch + P - 1) / P;
                    const int64_t slots = (int64_t)r.sm_count * ctas;
                    const double total = t * (double)((nunits + slots - 1) / slots) + 3000.0;
                    if (!(total < best.total * 0.995)) continue;
                    KsCand c;
                    c.ok = true;
                    c.dmma = 1;
                    c.single = 1;
                    c.total = total;
                    c.unit = t;
                    c.P = P;
                    c.S = S;
                    c.W = W;
                    c.ctas = ctas;
                    c.a_bytes = a_bytes;
                    c.b_bytes = b_bytes;
                    c.a_pitch = da;
                    c.b_pitch = db;
                    c.ms.s[0] = {8 * wm, tm};
                    c.ms.n = 1;
                    c.ns.s[0] = {8 * wn, tn};
                    c.ns.n = 1;
                    c.memops = (int64_t)tiles * (8 * wm + 8 * wn) * K + 2 * M * N;
                    c.ncls = 1;
                    c.cls[0] = IaatClass{catalog_code(IAAT_FAM_DMMA, 8 * wm, 8 * wn), 0, W, tiles, tm, 0, 8 * wm, 0,
                                         8 * wn, tn, 0, 0};
                    best = c;
                }
            }
        }
    if (!best.ok) return false;
    Plan &pl = out;
    pl = Plan();
    pl.ks = 1;
    IaatKsParams &k = pl.ksp;
    std::memset(&k, 0, sizeof k);
    k.sC = r.sC;
    k.batch = r.batch;
    k.nunits = (r.batch + best.P - 1) / best.P;
    k.M = (int)M;
    k.N = (int)N;
    k.K = (int)K;
    k.ldc = (int)r.ldc;
    k.P = best.P;
    k.S = best.S;
    k.kc = kc;
    k.nchunks = nchunks;
    k.n_compute_warps = best.W;
    k.a_pitch = best.a_pitch;
    k.b_pitch = best.b_pitch;
    k.a_bytes = best.a_bytes;
    k.b_bytes = best.b_bytes;
    k.a_tx = (int)((int64_t)best.P * (AK ? M * 128 : (int64_t)kc * best.a_pitch * 8));
    k.b_tx = (int)((int64_t)best.P * (BK ? N * 128 : (int64_t)kc * best.b_pitch * 8));
    k.stage_bytes = best.a_bytes + best.b_bytes;
    k.beta_zero = r.beta_zero;
    k.c_vec = 1;
    k.cplx = 1;
    k.c_elt = 16;
    k.nclasses = 1;
    k.cls[0] = best.cls[0];
    // tensor maps on the real (re, im) view: dims in doubles, strides in bytes
    auto geo = [&](TmaGeo &g, int64_t rows, int64_t cols, int64_t ld, int64_t stride, bool kmaj, int pitch, int D) {
        g.dim[0] = (uint64_t)(2 * rows);
        g.dim[1] = (uint64_t)cols;
        g.dim[2] = (uint64_t)r.batch;
        g.stride[0] = (uint64_t)(ld * 16);
        g.stride[1] = (uint64_t)((r.batch > 1 ? stride : ld * cols) * 16);
        if (kmaj) {
            g.box[0] = 16;  // 8 complex
            g.box[1] = (uint32_t)D;
        } else {
            g.box[0] = (uint32_t)pitch;
            g.box[1] = (uint32_t)kc;
        }
        g.box[2] = (uint32_t)best.P;
        g.swizzle128 = kmaj ? 1 : 0;
    };
    geo(pl.tmA, rowsA, colsA, r.lda, r.sA, AK, best.a_pitch, (int)M);
    geo(pl.tmB, rowsB, colsB, r.ldb, r.sB, BK, best.b_pitch, (int)N);
    pl.family = IAAT_FAM_KS_DMMA;
    pl.single = 1;
    pl.ksd = 1;
    pl.vec = 1;
    pl.ctas = best.ctas;
    pl.grid = (int)std::min<int64_t>(k.nunits, (int64_t)r.sm_count * best.ctas);
    pl.block = (best.W + 1) * 32;
    pl.smem = IAAT_KS_BAR_BYTES + 1024 + best.S * k.stage_bytes;
    pl.nm = 1;
    pl.nn = 1;
    pl.mstrip[0] = best.ms.s[0];
    pl.nstrip[0] = best.ns.s[0];
    pl.memops = best.memops;
    pl.est_cycles = best.unit;
    pl.est_total = best.total;
    pl.status = 0;
    return true;
}

bool plan_ks(const PlanRequest &r, const Knobs &kn, Plan &out)
{
    if (r.ptr_array || r.dtype == 2) return false;  // complex fp32: slab family only
    if (r.dtype == 3) return plan_ks_zdmma(r, kn, out);  // complex fp64: K-streamed DMMA (ZGEMM)
    const int elt = r.dtype == 0 ? 4 : 8;
    const int vw = 16 / elt, KU = vw, kc = 128 / elt;
    const int tidx = r.transA * 2 + r.transB;
    const int64_t M = r.M, N = r.N, K = r.K;
    const bool AK = r.transA == 1, BK = r.transB == 0;
    const int64_t rowsA = AK ? K : M, colsA = AK ? M : K, rowsB = BK ? K : N, colsB = BK ? N : K;
    auto al16 = [&](int64_t el) { return (el * elt) % 16 == 0; };
    if (M > 256 || N > 256 || K < 1) return false;
    if (r.batch > 1 && (r.sA < r.lda * colsA || r.sB < r.ldb * colsB)) return false;  // (0 = broadcast: slab family)
    // TMA boxes need 16-byte aligned bases, ld's and strides; otherwise the
    // same stages are filled element-wise with cp.async (LDGSTS mode, FMA tiles)
    bool tma_ok = r.align % 16 == 0 && al16(r.lda) && al16(r.ldb);
    if (r.batch > 1 && (!al16(r.sA) || !al16(r.sB) || r.sA * elt >= (int64_t)1 << 40 || r.sB * elt >= (int64_t)1 << 40))
        tma_ok = false;
    const int ldgsts = tma_ok ? 0 : 1;
    if (ldgsts && kn.fam == IAAT_FAM_KS_DMMA) return false;  // DMMA steps read the zero fill past K
    if (r.batch >= ((int64_t)1 << 31)) return false;
    const int a_pitch = AK ? kc : (int)round_up(M, vw), b_pitch = BK ? kc : (int)round_up(N, vw);
    if (a_pitch > 256 || b_pitch > 256) return false;
    const bool c_vec = r.align % 16 == 0 && al16(r.ldc) && (r.batch <= 1 || al16(r.sC));
    const double hbm_per_problem = (double)(M * K + K * N + M * N * (r.beta_zero ? 1 : 2)) * elt;
    const int nchunks = (int)((K + kc - 1) / kc);

    static const int kMaps[8] = {-2, -1, 1, 2, 4, 8, 16, 32};
    auto msplits = splits((int)M, 8, vw);
    auto nsplits = splits((int)N, 8, vw);
    KsCand best;
    const bool want_dmma = kn.fam == IAAT_FAM_KS_DMMA;
    for (const auto &ms : msplits)
        for (const auto &ns : nsplits) {
            if (want_dmma) break;
            if (kn.mr && (ms.s[0].size != kn.mr || ns.s[0].size != kn.nr)) continue;
            struct Cl {
                int mr, nr, tm, tn, rb, cb;
                double instr[8], wf[8];
                bool ok[8];
            } cl[4];
            int ncl = 0;
            bool avail = true;
            // one class covering C -> its single-class kernel if generated;
            // otherwise every class must be in the multi-class kernel
            const bool one = ms.n == 1 && ns.n == 1;
            int single = one && catalog_has(r.dtype, tidx, IAAT_FAM_KS1_FMA, ms.s[0].size, ns.s[0].size) ? 1 : 0;
            if (kn.fam == IAAT_FAM_KSU_FMA) {
                // uniform-phase kernels: one class whose K-major tile counts are multiples of 8
                if (!one || !catalog_has(r.dtype, tidx, IAAT_FAM_KSU_FMA, ms.s[0].size, ns.s[0].size)) continue;
                if ((AK && ms.s[0].count % 8) || (BK && ns.s[0].count % 8)) continue;
                single = 2;
            }
            int64_t memops = 2 * M * N;
            int rb = 0;
            for (int a = 0; a < ms.n && avail; ++a) {
                int cb = 0;
                for (int b = 0; b < ns.n; ++b) {
                    const int mr = ms.s[a].size, nr = ns.s[b].size;
                    if (single == 0 && !catalog_has(r.dtype, tidx, IAAT_FAM_KS_FMA, mr, nr)) {
                        avail = false;
                        break;
                    }
                    Cl &q = cl[ncl++];
                    q.mr = mr;
                    q.nr = nr;
                    q.tm = ms.s[a].count;
                    q.tn = ns.s[b].count;
                    q.rb = rb;
                    q.cb = cb;
                    for (int m = 0; m < 8; ++m) {
                        const int map = kMaps[m];
                        q.ok[m] = true;
                        if (kn.order >= 0 && !((kn.order == 0 && map == -2) || (kn.order == 1 && map == -1) ||
                                               (kn.order >= 2 && map == kn.order - 1)))
                            q.ok[m] = false;
                        Lanes L = lane_map(map, q.tm * q.tn, q.tm, q.tn);
                        if (map > 0 && (L.active < 24 || q.tm * q.tn < 32)) q.ok[m] = false;
                        if (!q.ok[m]) continue;
                        ks_class_cost(r, elt, mr, nr, L, rb, cb, q.tm, q.tn, a_pitch, b_pitch, kc, q.instr[m],
                                      q.wf[m]);
                    }
                    memops += (int64_t)q.tm * q.tn * (mr + nr) * K;
                    cb += ns.s[b].size * ns.s[b].count;
                }
                rb += ms.s[a].size * ms.s[a].count;
            }
            if (!avail) continue;
            for (int ctas = 1; ctas <= 4; ++ctas) {
                if (kn.ctas && ctas != kn.ctas) continue;
                // 128 registers per thread -> at most 16 resident warps per SM
                // (4 per SM sub-partition), producers included
                const int wmax = std::min(IAAT_MAX_THREADS / 32, 16 / ctas) - 1;
                if (wmax < 1) continue;
                const int smem_cta = (int)std::min<int64_t>(IAAT_SMEM_LIMIT, 228 * 1024 / ctas - 1024);
                for (int P = 1; P <= 64; ++P) {
                    if (kn.p && P != kn.p) continue;
                    if (P > 1 && (int64_t)(P - 1) * r.sm_count * ctas >= r.batch) break;
                    int W = 0;
                    double instr = 0, wf = 0;
                    int pick[4];
                    bool fits = true;
                    for (int q = 0; q < ncl; ++q) {
                        double bk = 1e300;
                        pick[q] = -1;
                        for (int m = 0; m < 8; ++m) {
                            if (!cl[q].ok[m]) continue;
                            const int w = class_warps(kMaps[m], P, cl[q].tm * cl[q].tn, cl[q].tm, cl[q].tn);
                            if (W + w > wmax) continue;  // mapping must leave room in the CTA
                            const double k = w * std::max(cl[q].instr[m] / kIssuePerClk, cl[q].wf[m] / kSmemPerClk);
                            if (k < bk * 0.999) {
                                bk = k;
                                pick[q] = m;
                            }
                        }
                        if (pick[q] < 0) {
                            fits = false;
                            break;
                        }
                        const int w = class_warps(kMaps[pick[q]], P, cl[q].tm * cl[q].tn, cl[q].tm, cl[q].tn);
                        W += w;
                        instr += w * cl[q].instr[pick[q]];
                        wf += w * cl[q].wf[pick[q]];
                    }
                    if (!fits) continue;
                    if (W > wmax) break;
                    const int a_bytes = (int)round_up((int64_t)P * (AK ? M * 128 : (int64_t)kc * a_pitch * elt), 1024);
                    const int b_bytes = (int)round_up((int64_t)P * (BK ? N * 128 : (int64_t)kc * b_pitch * elt), 1024);
                    const int stage = a_bytes + b_bytes;
                    int S = std::min(IAAT_KS_MAX_STAGES, (smem_cta - IAAT_KS_BAR_BYTES - 1024) / stage);
                    if (kn.s > 0) S = std::min(S, kn.s);
                    if (S < 2) continue;
                    // one round: every resident CTA finishes one unit
                    const double nblk = (double)K / KU;
                    const double t_hbm = ctas * P * hbm_per_problem / kHbmBytesPerClk;
                    const double rate = std::min(kIssuePerClk, kIssuePerWarp * 1.5 * ctas * W);
                    const double epi = (double)P * M * N * (r.beta_zero ? 2 : 4) / 32.0;
                    const double t_issue = ctas * (instr * nblk + epi + W * nchunks * 12.0) / rate;
                    const double t_smem = ctas * wf * nblk / kSmemPerClk;
                    const double t_comp = std::max(t_issue, t_smem);
                    // latency to fill: S stages must cover ~kLoadLatency of the ring
                    const double t_lat = kLoadLatency * nchunks / std::max(1, S - 1) / ctas;
                    const double t = std::max(std::max(t_hbm, t_comp), t_lat) + 0.15 * std::min(t_hbm, t_comp) + 300.0;
                    const int64_t nunits = (r.batch + P - 1) / P;
                    const int64_t slots = (int64_t)r.sm_count * ctas;
                    const double total = t * (double)((nunits + slots - 1) / slots) + 3000.0;
                    if (!(total < best.total * 0.995 || (!(best.total < total * 0.995) && memops < best.memops)))
                        continue;
                    KsCand c;
                    c.ok = true;
                    c.single = single;
                    c.total = total;
                    c.unit = t;
                    c.P = P;
                    c.S = S;
                    c.W = W;
                    c.ctas = ctas;
                    c.a_bytes = a_bytes;
                    c.b_bytes = b_bytes;
                    c.a_pitch = a_pitch;
                    c.b_pitch = b_pitch;
                    c.ms = ms;
                    c.ns = ns;
                    c.memops = memops;
                    c.ncls = ncl;
                    int wb = 0;
                    for (int q = 0; q < ncl; ++q) {
                        const int map = kMaps[pick[q]];
                        const int w = class_warps(map, P, cl[q].tm * cl[q].tn, cl[q].tm, cl[q].tn);
                        c.cls[q] = IaatClass{catalog_code(IAAT_FAM_FMA, cl[q].mr, cl[q].nr), wb, wb + w,
                                             cl[q].tm * cl[q].tn, cl[q].tm, cl[q].rb, cl[q].mr, cl[q].cb, cl[q].nr,
                                             cl[q].tn, map == -1 ? 1 : 0, map > 0 ? map : 0};
                        wb += w;
                    }
                    best = c;
                }
            }
        }

    // ---------------- fp64 DMMA warp tiles (one class: (8 wm) x (8 wn) blocks, one per warp)
    if (want_dmma && r.dtype == 1 && M % 8 == 0 && N % 8 == 0) {
        // MN-major pitch = 4 (mod 16) doubles: the 4 k-rows a half-warp reads
        // fall into 4 different 32-byte bank windows
        auto dpitch = [](int64_t D) { int64_t q = D; while (q % 16 != 4) ++q; return (int)q; };
        const int da = AK ? kc : dpitch(M), db = BK ? kc : dpitch(N);
        for (int wm = 1; wm <= 7; ++wm)  // the catalog decides which (wm, wn) exist
            for (int wn = 1; wn <= 7; ++wn) {
                if ((M / 8) % wm || (N / 8) % wn) continue;
                if (kn.mr && (8 * wm != kn.mr || 8 * wn != kn.nr)) continue;
                if (!catalog_has(1, tidx, IAAT_FAM_KS_DMMA, 8 * wm, 8 * wn)) continue;
                const int tm = (int)(M / (8 * wm)), tn = (int)(N / (8 * wn)), tiles = tm * tn;
                for (int ctas = 1; ctas <= 3; ++ctas) {
                    if (kn.ctas && ctas != kn.ctas) continue;
                    const int wmax = IAAT_KSD_THREADS(wm, wn) / 32 / ctas - 1;
                    const int smem_cta = (int)std::min<int64_t>(IAAT_SMEM_LIMIT, 228 * 1024 / ctas - 1024);
                    for (int P = 1; P * tiles <= wmax; ++P) {
                        if (kn.p && P != kn.p) continue;
                        if (P > 1 && (int64_t)(P - 1) * r.sm_count * ctas >= r.batch) break;
                        const int W = P * tiles;
                        const int a_bytes = (int)round_up((int64_t)P * (AK ? M * 128 : (int64_t)kc * da * 8), 1024);
                        const int b_bytes = (int)round_up((int64_t)P * (BK ? N * 128 : (int64_t)kc * db * 8), 1024);
                        const int stage = a_bytes + b_bytes;
                        int S = std::min(IAAT_KS_MAX_STAGES, (smem_cta - IAAT_KS_BAR_BYTES - 1024) / stage);
                        if (kn.s > 0) S = std::min(S, kn.s);
                        if (S < 2) continue;
                        const double t_hbm = ctas * P * hbm_per_problem / kHbmBytesPerClk;
                        const double t_dmma = ctas * (double)P * M * N * K / kDfmaPerClk;
                        const double steps = (double)K / 4;
                        const double wf = ctas * W * steps * (wm + wn) * 3.0;  // LDS.64: 2 wavefronts, K-major up to 4
                        const double issue = ctas * W * steps * (wm * wn + (wm + wn) * 2 + 2) / kIssuePerClk;
                        const double t_lat = kLoadLatency * nchunks / std::max(1, S - 1) / ctas;
                        const double t_comp = std::max(std::max(t_dmma, wf / kSmemPerClk), issue);
                        const double t = std::max(std::max(t_hbm, t_comp), t_lat) + 0.15 * std::min(t_hbm, t_comp) + 300.0;
                        const int64_t nunits = (r.batch + P - 1) / P;
                        const int64_t slots = (int64_t)r.sm_count * ctas;
                        const double total = t * (double)((nunits + slots - 1) / slots) + 3000.0;
                        if (!(total < best.total * 0.995)) continue;
                        KsCand c;
                        c.ok = true;
                        c.dmma = 1;
                        c.single = 1;
                        c.total = total;
                        c.unit = t;
                        c.P = P;
                        c.S = S;
                        c.W = W;
                        c.ctas = ctas;
                        c.a_bytes = a_bytes;
                        c.b_bytes = b_bytes;
                        c.a_pitch = da;
                        c.b_pitch = db;
                        c.ms.s[0] = {8 * wm, tm};
                        c.ms.n = 1;
                        c.ns.s[0] = {8 * wn, tn};
                        c.ns.n = 1;
                        c.memops = (int64_t)tiles * (8 * wm + 8 * wn) * K + 2 * M * N;
                        c.ncls = 1;
                        c.cls[0] = IaatClass{catalog_code(IAAT_FAM_DMMA, 8 * wm, 8 * wn), 0, W, tiles, tm, 0, 8 * wm,
                                             0, 8 * wn, tn, 0, 0};
                        best = c;
                    }
                }
            }
    }
    if (!best.ok) return false;
    Plan &pl = out;
    pl = Plan();
    pl.ks = 1;
    IaatKsParams &k = pl.ksp;
    std::memset(&k, 0, sizeof k);
    k.sC = r.sC;
    k.batch = r.batch;
    k.nunits = (r.batch + best.P - 1) / best.P;
    k.M = (int)M;
    k.N = (int)N;
    k.K = (int)K;
    k.ldc = (int)r.ldc;
    k.P = best.P;
    k.S = best.S;
    k.kc = kc;
    k.nchunks = nchunks;
    k.n_compute_warps = best.W;
    k.a_pitch = best.a_pitch;
    k.b_pitch = best.b_pitch;
    k.a_bytes = best.a_bytes;
    k.b_bytes = best.b_bytes;
    k.a_tx = (int)((int64_t)best.P * (AK ? M * kc : (int64_t)kc * best.a_pitch) * elt);
    k.b_tx = (int)((int64_t)best.P * (BK ? N * kc : (int64_t)kc * best.b_pitch) * elt);
    k.stage_bytes = best.a_bytes + best.b_bytes;
    k.beta_zero = r.beta_zero;
    k.c_vec = c_vec ? 1 : 0;
    k.ldgsts = ldgsts;
    k.c_elt = elt;
    k.sA = r.sA;
    k.sB = r.sB;
    k.lda = (int)r.lda;
    k.ldb = (int)r.ldb;
    k.nclasses = best.ncls;
    for (int q = 0; q < best.ncls; ++q) k.cls[q] = best.cls[q];
    auto geo = [&](TmaGeo &g, int64_t rows, int64_t cols, int64_t ld, int64_t stride, bool kmaj, int pitch, int D) {
        g.dim[0] = (uint64_t)rows;
        g.dim[1] = (uint64_t)cols;
        g.dim[2] = (uint64_t)r.batch;
        g.stride[0] = (uint64_t)(ld * elt);
        g.stride[1] = (uint64_t)((r.batch > 1 ? stride : ld * cols) * elt);
        if (kmaj) {
            g.box[0] = (uint32_t)kc;
            g.box[1] = (uint32_t)D;
        } else {
            g.box[0] = (uint32_t)pitch;
            g.box[1] = (uint32_t)kc;
        }
        g.box[2] = (uint32_t)best.P;
        g.swizzle128 = kmaj ? 1 : 0;
    };
    geo(pl.tmA, rowsA, colsA, r.lda, r.sA, AK, best.a_pitch, (int)M);
    geo(pl.tmB, rowsB, colsB, r.ldb, r.sB, BK, best.b_pitch, (int)N);
    pl.family = best.dmma ? IAAT_FAM_KS_DMMA : IAAT_FAM_KS_FMA;
    pl.single = best.single;
    pl.ksd = best.dmma;
    pl.vec = 1;
    pl.ctas = best.ctas;
    pl.grid = (int)std::min<int64_t>(k.nunits, (int64_t)r.sm_count * best.ctas);
    pl.block = (best.W + 1) * 32;
    pl.smem = IAAT_KS_BAR_BYTES + 1024 + best.S * k.stage_bytes;
    pl.nm = best.ms.n;
    pl.nn = best.ns.n;
    for (int i = 0; i < 2; ++i) {
        pl.mstrip[i] = best.ms.s[i];
        pl.nstrip[i] = best.ns.s[i];
    }
    pl.memops = best.memops;
    pl.est_cycles = best.unit;
    pl.est_total = best.total;
    pl.status = 0;
    return true;
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
        p.status, r.dtype == 0 ? "f32" : r.dtype == 1 ? "f64" : r.dtype == 2 ? "c32" : "c64", r.transA ? 'T' : 'N', r.transB ? 'T' : 'N', (long long)r.M,
        (long long)r.N, (long long)r.K);
    if (p.status != 0) {
        s += "\"classes\": []}";
        return s;
    }
    const IaatKParams &k = p.kp;
    add("\"tuned\": %d, ", p.tuned);
    if (p.ksg == 2) {
        const IaatKsgParams &q = p.kgp;
        const IaatKsgsCatalogEntry &e = kKsgsCatalog[p.kg_entry];
        add("\"family\": \"ksgs\", \"entry\": %d, \"mr\": %d, \"nr\": %d, \"lane_rows\": %d, \"groups\": %d, "
            "\"warps_per_group\": %d, \"Mv\": %d, \"Nv\": %d, \"P\": %d, \"S\": %d, \"a_bytes\": %d, "
            "\"b_bytes\": %d, \"c_bytes\": %d, \"grid\": %d, \"block\": %d, \"smem\": %d, \"nunits\": %lld, "
            "\"est\": %.0f, \"memops\": %lld, ",
            p.kg_entry, e.mr, e.nr, e.lr, e.g, e.w, q.Mv, q.Nv, q.P, q.S, q.a_bytes, q.b_bytes, q.c_bytes, p.grid,
            p.block, p.smem, (long long)q.nunits, p.est_total, (long long)p.memops);
        s += "\"classes\": []}";
        return s;
    }
    if (p.ksg) {
        const IaatKsgParams &q = p.kgp;
        const IaatKsgCatalogEntry &e = kKsgCatalog[p.kg_entry];
        add("\"family\": \"ksg\", \"entry\": %d, \"mr\": %d, \"nr\": %d, \"lane_rows\": %d, \"kc\": %d, "
            "\"ku\": %d, \"groups\": %d, \"warps_per_group\": %d, \"Mv\": %d, \"Nv\": %d, \"P\": %d, \"S\": %d, "
            "\"c_pitch\": %d, \"grid\": %d, \"block\": %d, \"smem\": %d, \"nunits\": %lld, \"est\": %.0f, "
            "\"memops\": %lld, \"pairv\": %d, \"stage_bytes\": %d, \"c_bytes\": %d, ",
            p.kg_entry, e.mr, e.nr, e.lr, e.kc, e.ku, e.g, e.w, q.Mv, q.Nv, q.P, q.S, q.c_pitch, p.grid, p.block,
            p.smem, (long long)q.nunits, p.est_total, (long long)p.memops, q.pairv, q.stage_bytes, q.c_bytes);
        s += "\"classes\": []}";
        return s;
    }
    const int ncls = p.ks ? p.ksp.nclasses : k.nclasses;
    const IaatClass *cls = p.ks ? p.ksp.cls : k.cls;
    if (p.ks) {
        const IaatKsParams &q = p.ksp;
        add("\"family\": \"%s\", \"vec\": %d, \"P\": %d, \"S\": %d, \"compute_warps\": %d, "
            "\"ctas_per_sm\": %d, \"grid\": %d, \"block\": %d, \"smem\": %d, \"ngroups\": %lld, ",
            p.ksd ? "ks_dmma" : p.single == 2 ? "ksu_fma" : p.single ? "ks1_fma" : "ks_fma", p.vec, q.P, q.S, q.n_compute_warps, p.ctas, p.grid, p.block, p.smem,
            (long long)q.nunits);
        add("\"kc\": %d, \"nchunks\": %d, \"a_bytes\": %d, \"b_bytes\": %d, \"a_pitch\": %d, \"b_pitch\": %d, "
            "\"a_swizzle128\": %d, \"b_swizzle128\": %d, \"c_vec\": %d, \"ldgsts\": %d, ",
            q.kc, q.nchunks, q.a_bytes, q.b_bytes, q.a_pitch, q.b_pitch, p.tmA.swizzle128, p.tmB.swizzle128, q.c_vec,
            q.ldgsts);
    } else {
        add("\"family\": \"%s\", \"vec\": %d, \"P\": %d, \"S\": %d, \"compute_warps\": %d, \"ctas_per_sm\": %d, "
            "\"grid\": %d, \"block\": %d, \"smem\": %d, \"ngroups\": %lld, ",
            p.family == IAAT_FAM_DMMA ? "dmma" : "fma", p.vec, k.P, k.S, k.n_compute_warps, p.ctas, p.grid, p.block,
            p.smem, (long long)k.ngroups);
        add("\"stage_a\": \"%s\", \"stage_b\": \"%s\", \"stage_c\": \"%s\", \"cap_a\": %d, \"cap_b\": %d, "
            "\"cap_c\": %d, \"c_in_smem\": %d, \"prefetch_c\": %d, ",
            k.modeA ? "perprob" : "slab", k.modeB ? "perprob" : "slab", k.modeC ? "perprob" : "slab", k.capA,
            k.capB, k.capC, k.c_in_smem, k.prefetch_c);
    }
    add("\"m_strips\": [");
    for (int i = 0; i < p.nm; ++i) add("%s[%d, %d]", i ? ", " : "", p.mstrip[i].size, p.mstrip[i].count);
    add("], \"n_strips\": [");
    for (int i = 0; i < p.nn; ++i) add("%s[%d, %d]", i ? ", " : "", p.nstrip[i].size, p.nstrip[i].count);
    add("], \"memops\": %lld, \"est_cycles_per_group\": %.1f, \"est_cycles_total\": %.1f, \"classes\": [",
        (long long)p.memops, p.est_cycles, p.est_total);
    for (int q = 0; q < ncls; ++q) {
        const IaatClass &c = cls[q];
        add("%s{\"code\": %d, \"mr\": %d, \"nr\": %d, \"tiles\": %d, \"tm\": %d, \"row_base\": %d, "
            "\"col_base\": %d, \"warp_begin\": %d, \"warp_end\": %d, \"colfast\": %d, \"bm\": %d}",
            q ? ", " : "", c.code, c.mr, c.nr, c.tiles, c.tm, c.row_base, c.col_base, c.warp_begin,
            c.warp_end, c.colfast, c.bm);
    }
    s += "]}";
    return s;
}


// ============================================================================
// Paper-faithful tiling mode (an ablation baseline for the GPU
// planner, host only).  The SGEMM_NN kernel catalog of Table I (PAPER.md:94,
// the NN column of the SGEMM row) and the run-time tile algorithm of Sec.
// V-A (Alg. 2) with its memops cost "(m_0 + n_0 + ... +
// m_a + n_a) K + 2mn".
//   mode 0: Alg. 2 traced literally, with the readings of DESIGN.md A14:
//           ExtendTo8/16(m1) regroup the 4-high strips into 8-/16-high ones
//           (remainder stays 4); "tile N by m8[] / m16[]" = TileSingleDim(N,
//           widths allowed for that height); TileSingleDim is greedy
//           largest-first and averages the last two pieces when the
//           remainder is below half the largest width (the threshold of
//           PAPER.md:319 is unstated).
//   mode 1: the exact optimum over Table I: row strips of catalog heights,
//           each strip tiled in N by its widest allowed width (a strip of
//           height h costs ceil(N / w_max(h)) * h + N), dynamic programming
//           over M -- the decomposition behind Fig. 2's 72K + 450 for 15 x 15
//           (PAPER.md:337).
// ============================================================================
namespace paper {

struct Piece {
    int dim, nums;
};
struct StripPlan {
    int h, count;
    std::vector<Piece> n;  // widths of one strip
};

// Table I, SGEMM NN: m_c -> the largest n_c (every n_c from 1 up is generated)
int nmax_nn(int mc)
{
    switch (mc) {
    case 16: return 4;
    case 12: return 6;
    case 8: return 8;
    case 4: case 3: case 2: case 1: return 13;
    }
    return 0;
}

// TileSingleDim(D, sizes): (dim, nums) pairs, largest first
std::vector<Piece> tile_single_dim(int D, const std::vector<int> &sizes)
{
    int big = 0;
    for (int s : sizes) big = std::max(big, s);
    std::vector<Piece> out;
    if (D <= 0 || big <= 0) return out;
    const int q = D / big, r = D % big;
    if (q > 0) out.push_back({big, q});
    if (r > 0) {
        if (q > 0 && 2 * r < big) {
            // average the last two pieces: big + r -> two near-equal widths
            const int a = (big + r + 1) / 2, b = (big + r) / 2;
            if (out.back().nums == 1) out.pop_back(); else out.back().nums -= 1;
            out.push_back({a, 1});
            if (b > 0) out.push_back({b, 1});
        } else {
            out.push_back({r, 1});
        }
    }
    return out;
}

std::vector<int> range1(int hi)
{
    std::vector<int> v;
    for (int i = 1; i <= hi; ++i) v.push_back(i);
    return v;
}

int64_t strips_cost(const std::vector<StripPlan> &s)
{
    int64_t c = 0;
    for (const auto &p : s)
        for (const auto &w : p.n) c += (int64_t)p.count * w.nums * (p.h + w.dim);
    return c;
}

// ExtendTo8 / ExtendTo16 of m1 = (4, q): regroup 4-strips into e-high strips
std::vector<StripPlan> extend(int q, int e, int N)
{
    std::vector<StripPlan> v;
    const int per = e / 4, big = q / per, rem = q % per;
    if (big > 0) v.push_back({e, big, tile_single_dim(N, range1(nmax_nn(e)))});
    if (rem > 0) v.push_back({4, rem, tile_single_dim(N, range1(nmax_nn(4)))});
    return v;
}

std::vector<StripPlan> alg2_literal(int M, int N)
{
    std::vector<StripPlan> s;
    if (N <= 13) {
        // lines 1-7: n_c = N, m_1 the largest m_c whose kernel has n_c = N
        int m1 = 1;
        for (int mc : {16, 12, 8, 4, 3, 2, 1})
            if (nmax_nn(mc) >= N && mc <= M) {
                m1 = mc;
                break;
            }
        const int I = M / m1;
        s.push_back({m1, I, {{N, 1}}});
        // line 5 appends (M - m_1 I, 1); a remainder with no kernel of its
        // own height (5, 6, 7, 9, 10, 11, 13-15) is split into Table I
        // heights largest-first (reading A14)
        for (int rem = M - m1 * I; rem > 0;) {
            int h = 1;
            for (int mc : {16, 12, 8, 4, 3, 2, 1})
                if (mc <= rem && nmax_nn(mc) >= N) {
                    h = mc;
                    break;
                }
            s.push_back({h, 1, {{N, 1}}});
            rem -= h;
        }
        return s;
    }
    const std::vector<int> w13 = range1(13), w8 = range1(8), w6 = range1(6);
    if (M < 8) {
        for (const Piece &p : tile_single_dim(M, {1, 2, 3, 4})) s.push_back({p.dim, p.nums, tile_single_dim(N, w13)});
    } else if (M == 9) {
        for (int h : {4, 3, 2}) s.push_back({h, 1, tile_single_dim(N, w13)});
    } else if (M < 12) {
        s.push_back({8, 1, tile_single_dim(N, w8)});
        if (M > 8) s.push_back({M - 8, 1, tile_single_dim(N, w13)});  // (M-8, 1) is empty at M == 8 (reading A14)
    } else if (M == 12) {
        s.push_back({12, 1, tile_single_dim(N, w6)});
    } else {
        int q = M / 4;
        std::vector<StripPlan> m2;
        if (M - 4 * q == 1) {
            q -= 1;
            m2.push_back({3, 1, tile_single_dim(N, w8)});
            m2.push_back({2, 1, tile_single_dim(N, w13)});
        } else if (M - 4 * q > 0) {
            m2.push_back({M - 4 * q, 1, tile_single_dim(N, w13)});
        }
        std::vector<StripPlan> b8 = extend(q, 8, N), b16 = extend(q, 16, N);
        s = strips_cost(b16) < strips_cost(b8) ? b16 : b8;  // CompareLessMemops
        for (auto &p : m2) s.push_back(p);
    }
    return s;
}

std::vector<StripPlan> optimal(int M, int N)
{
    const int H[] = {16, 12, 8, 4, 3, 2, 1};
    std::vector<int64_t> best(M + 1, (int64_t)1 << 60);
    std::vector<int> pick(M + 1, 0);
    best[0] = 0;
    for (int m = 1; m <= M; ++m)
        for (int h : H) {
            if (h > m) continue;
            const int64_t c = best[m - h] + (int64_t)((N + nmax_nn(h) - 1) / nmax_nn(h)) * h + N;
            if (c < best[m]) {  // ties: the first (larger) height wins
                best[m] = c;
                pick[m] = h;
            }
        }
    std::vector<StripPlan> s;
    for (int m = M; m > 0; m -= pick[m]) {
        const int h = pick[m], w = nmax_nn(h);
        std::vector<Piece> n;
        if (N / w) n.push_back({w, N / w});
        if (N % w) n.push_back({N % w, 1});
        if (!s.empty() && s.back().h == h) s.back().count += 1;
        else s.push_back({h, 1, n});
    }
    return s;
}

}  // namespace paper

std::string paper_tile_json(int mode, int M, int N)
{
    std::vector<paper::StripPlan> s = mode == 0 ? paper::alg2_literal(M, N) : paper::optimal(M, N);
    std::string j = "{\"mode\": \"";
    j += mode == 0 ? "alg2_literal" : "table1_optimal";
    j += "\", \"strips\": [";
    char buf[128];
    for (size_t i = 0; i < s.size(); ++i) {
        std::snprintf(buf, sizeof buf, "%s{\"h\": %d, \"count\": %d, \"n\": [", i ? ", " : "", s[i].h, s[i].count);
        j += buf;
        for (size_t k = 0; k < s[i].n.size(); ++k) {
            std::snprintf(buf, sizeof buf, "%s[%d, %d]", k ? ", " : "", s[i].n[k].dim, s[i].n[k].nums);
            j += buf;
        }
        j += "]}";
    }
    std::snprintf(buf, sizeof buf, "], \"memops_k_coeff\": %lld, \"memops_const\": %lld}",
                  (long long)paper::strips_cost(s), (long long)2 * M * N);
    j += buf;
    return j;
}

}  // namespace iaat
