"""Run-time planner (csrc/planner.cpp) through the host-only C ABI entry
iaat_plan_describe -- CPU only.

Invariants the kernels rely on: every plan's tile classes cover
the M x N index set exactly once with catalog tiles ("each block
has the same size as one of the generated kernels"), warps are partitioned
into contiguous warp-uniform class ranges, vector-capable classes start on a
vector boundary, shared memory fits, and planning is deterministic.
"""
import itertools

import numpy as np
import pytest

from paper_2208_09822_b200 import iaat

CAT = iaat.iaat_catalog_describe()
TRANS = ["NN", "NT", "TN", "TT"]


def catalog_set():
    s = set()
    for e in CAT:
        s.add((e["family"], e["dtype"], e["trans"], e["mr"], e["nr"]))
    return s


CATSET = catalog_set()


def plan(dt, tr, M, N, K, batch=10000, beta0=False, align=256, pad=0):
    ra, ca = (M, K) if tr[0] == "N" else (K, M)
    rb, cb = (K, N) if tr[1] == "N" else (N, K)
    lda, ldb, ldc = ra + pad, rb + pad, M + pad
    return iaat.iaat_plan_describe(dt, tr[0], tr[1], M, N, K, lda, lda * ca, ldb, ldb * cb, ldc, ldc * N, batch,
                                   beta0, False, align, 148)


KSG = {e["index"]: e for e in CAT if e["family"] == "ksg"}


KSGS = {e["index"]: e for e in CAT if e["family"] == "ksgs"}


def check_ksgs_plan(p, tr, M, N):
    e = KSGS[p["entry"]]
    br, bc = e["lr"] * e["mr"], (32 // e["lr"]) * e["nr"]
    assert e["trans"] == tr and p["Mv"] % br == 0 and p["Nv"] % bc == 0
    assert M <= p["Mv"] < M + br and N <= p["Nv"] < N + bc
    assert (p["Mv"] // br) * (p["Nv"] // bc) * p["P"] == e["w"]
    assert p["smem"] <= 227 * 1024 and p["S"] >= 1
    # one ring of S stages [A | B | C] shared by the groups, after the 1 KB barrier area
    assert p["smem"] >= 2048 + p["S"] * (p["a_bytes"] + p["b_bytes"] + p["c_bytes"])


def check_ksg_plan(p, tr, M, N):
    """ksg (csrc/iaat_ksg.cuh): one lane-grid class whose warp blocks tile the
    Mv x Nv problem exactly; Mv - M, Nv - N < one warp block (the copy
    engine's zero fill covers them, the TMA store clips them), whole
    problems per group, M on a 16-byte C granule, smem within the limit."""
    e = KSG[p["entry"]]
    assert e["trans"] == tr and (e["mr"], e["nr"], e["lr"]) == (p["mr"], p["nr"], p["lane_rows"])
    br, bc = e["lr"] * e["mr"], (32 // e["lr"]) * e["nr"]
    assert p["Mv"] % br == 0 and p["Nv"] % bc == 0
    assert M <= p["Mv"] < M + br and N <= p["Nv"] < N + bc
    wpp = (p["Mv"] // br) * (p["Nv"] // bc)
    assert wpp * p["P"] == e["w"]
    assert e["g"] * e["w"] in (8, 12) and p["block"] == 128 + 32 * e["g"] * e["w"]
    assert p["smem"] <= 227 * 1024 and 1 <= p["S"] <= 8
    r1k = lambda x: -(-x // 1024) * 1024  # noqa: E731
    P, kc = p["P"], e["kc"]
    if p["pairv"]:
        # column-pair boxes (n = 2 mod 4): packed even extents, C columns M
        # apart; MN-major boxes hold the packed columns, K-major ones two
        # unswizzled half boxes (even / odd columns) with rows of kc + 4
        assert M % 2 == 0 and N % 2 == 0 and p["c_pitch"] == M
        r128 = lambda x: -(-x // 128) * 128  # noqa: E731
        a = 2 * r128(P * p["Mv"] // 2 * (kc + 4) * 4) if tr[0] == "T" else r128(P * M * kc * 4)
        b = 2 * r128(P * p["Nv"] // 2 * (kc + 4) * 4) if tr[1] == "N" else r128(P * N * kc * 4)
        group = p["S"] * (a + b) + r128(P * p["Nv"] * M * 4)
        assert p["stage_bytes"] == a + b
    else:
        assert M % 4 == 0
        assert p["c_pitch"] >= p["Mv"] and p["c_pitch"] % 4 == 0
        # every group's ring (S stages of one A box and one B box) and C buffer fit
        group = p["S"] * (r1k(P * p["Mv"] * kc * 4) + r1k(P * p["Nv"] * kc * 4)) + r1k(P * p["Nv"] * p["c_pitch"] * 4)
    assert p["smem"] >= 2048 + e["g"] * group, (p, group)
    assert p["grid"] <= 148


def check_plan(p, dt, tr, M, N):
    assert p["status"] == 0, p
    if p.get("family") == "ksg":
        check_ksg_plan(p, tr, M, N)
        return
    if p.get("family") == "ksgs":
        check_ksgs_plan(p, tr, M, N)
        return
    cover = np.zeros((M, N), dtype=np.int32)
    dname = "f32" if dt == 0 else "f64"
    vw = 4 if dt == 0 else 2
    wprev = 0
    for c in p["classes"]:
        fam = p["family"]
        assert (fam, dname, tr, c["mr"], c["nr"]) in CATSET, c
        tm = c["tm"]
        tn = c["tiles"] // tm
        assert tm * tn == c["tiles"]
        for ti, tj in itertools.product(range(tm), range(tn)):
            r0 = c["row_base"] + ti * c["mr"]
            c0 = c["col_base"] + tj * c["nr"]
            cover[r0:r0 + c["mr"], c0:c0 + c["nr"]] += 1
            assert r0 + c["mr"] <= M and c0 + c["nr"] <= N
        # warp ranges contiguous and ordered
        assert c["warp_begin"] == wprev and c["warp_end"] > c["warp_begin"]
        wprev = c["warp_end"]
        if fam == "fma":
            assert p["P"] * c["tiles"] <= 32 * (c["warp_end"] - c["warp_begin"])
            if p["vec"]:
                if c["mr"] % vw == 0:
                    assert c["row_base"] % vw == 0
                if c["nr"] % vw == 0:
                    assert c["col_base"] % vw == 0
    assert np.all(cover == 1), "tiles do not cover C exactly once"
    assert wprev == p["compute_warps"] <= 15
    assert p["block"] == 32 * (p["compute_warps"] + 1)
    assert p["smem"] <= 227 * 1024
    if p["family"].startswith("ks"):
        # K-streamed: S-stage ring of K-chunks, 1024-byte aligned stages
        assert 2 <= p["S"] <= 12
        assert p["a_bytes"] % 1024 == 0 and p["b_bytes"] % 1024 == 0
        assert p["kc"] * (4 if dt == 0 else 8) == 128
        assert p["nchunks"] * p["kc"] >= p["K"] > (p["nchunks"] - 1) * p["kc"]
    else:
        assert 1 <= p["S"] <= 6
    assert p["grid"] <= 148 * p["ctas_per_sm"]


@pytest.mark.parametrize("tr", TRANS)
@pytest.mark.parametrize("dt", [0, 1])
def test_exact_cover_small(dt, tr):
    for M, N in itertools.product(range(1, 21), repeat=2):
        K = 7
        if tr == "TN" and M * N * K > 32768:
            continue
        check_plan(plan(dt, tr, M, N, K), dt, tr, M, N)


@pytest.mark.parametrize("tr", TRANS)
@pytest.mark.parametrize("dt", [0, 1])
def test_exact_cover_sampled_large(dt, tr):
    rng = np.random.default_rng(dt * 4 + TRANS.index(tr))
    lim = 32768 if tr == "TN" else 512000
    n = 0
    while n < 40:
        M, N, K = (int(x) for x in rng.integers(1, 81, size=3))
        if M * N * K > lim:
            continue
        n += 1
        for beta0 in (False, True):
            check_plan(plan(dt, tr, M, N, K, beta0=beta0), dt, tr, M, N)


def test_config_shapes_plan():
    for n in range(4, 81, 4):
        for tr in ("NN", "NT", "TT"):
            check_plan(plan(0, tr, n, n, n, batch=(256 << 20) // (12 * n * n)), 0, tr, n, n)
    for n in (8, 16, 32, 48, 64, 80):
        for tr in ("NN", "NT"):
            p = plan(1, tr, n, n, n, batch=2_000_000, beta0=True)
            check_plan(p, 1, tr, n, n)


def test_misaligned_and_padded_plans_disable_vectors():
    p = plan(0, "NN", 16, 16, 16, align=4)
    assert p["vec"] == 0
    p = plan(0, "NN", 16, 16, 16, pad=1)
    assert p["vec"] == 0
    p = plan(0, "NN", 16, 16, 16)
    assert p["vec"] == 1


def test_plan_deterministic():
    a = plan(0, "NT", 37, 53, 23)
    b = plan(0, "NT", 37, 53, 23)
    assert a == b


def test_small_batch_uses_all_sms():
    # config 1: 2000 problems -> at least 148 groups when possible
    p = plan(0, "NN", 16, 16, 16, batch=2000, beta0=True)
    assert p["P"] <= -(-2000 // 148)
    assert p["grid"] == p["ngroups"]


def test_memops_is_paper_cost():
    """memops = sum over tiles (m_i + n_i) K + 2MN."""
    for (M, N, K) in [(15, 15, 15), (64, 64, 64), (7, 80, 3)]:
        p = plan(0, "NN", M, N, K)
        if p["family"] == "ksg":  # lane tiles over the Mv x Nv tiling
            s = (p["Mv"] // p["mr"]) * (p["Nv"] // p["nr"]) * (p["mr"] + p["nr"])
        else:
            s = sum(c["tiles"] * (c["mr"] + c["nr"]) for c in p["classes"])
        assert p["memops"] == s * K + 2 * M * N


def test_catalog_register_budget():
    """Every catalog entry fits the generator's register budget (accumulators
    + live fragments, PAPER.md:217-235 register groups) -- the same budget the
    no-spill build check (tests/test_build.py) verifies."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "generate", os.path.join(os.path.dirname(iaat.__file__), "gen", "generate.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    for e in CAT:
        if e["family"] == "fma" and e["dtype"] in ("c32", "c64"):
            # complex micro-tiles: the generator's complex catalog
            assert (e["mr"], e["nr"]) in gen.cfma_tiles(e["dtype"], e["trans"])
        elif e["family"] == "fma":
            assert gen.fma_regs(e["dtype"], e["trans"], e["mr"], e["nr"]) <= gen.REG_BUDGET[e["dtype"]]
            assert 1 <= e["mr"] <= 8 and 1 <= e["nr"] <= 8
        elif e["family"] == "ksu_fma":
            assert e["dtype"] == "f32" and (e["mr"], e["nr"]) in gen.ksu_tiles(e["trans"])
        elif e["family"] == "ksg":
            # lane-grid register tiles (csrc/iaat_ksg.cuh): at most 128
            # accumulators, lanes lr x 32/lr, two or three consumer warpgroups
            assert e["dtype"] == "f32" and e["trans"] != "TN"
            assert e["mr"] * e["nr"] <= 128 and 32 % e["lr"] == 0
            assert e["g"] * e["w"] in (8, 12) and e["g"] <= 4 and e["kc"] in (16, 32) and e["ku"] in (1, 2, 4)
            assert tuple(e[k] for k in ("trans", "mr", "nr", "lr", "kc", "ku", "g", "w")) == gen.KSG_TILES[e["index"]]
        elif e["family"] == "ksgs":
            assert e["dtype"] == "f32" and e["mr"] * e["nr"] <= 100
            assert tuple(e[k] for k in ("trans", "mr", "nr", "lr", "g", "w")) == gen.KSGS_TILES[e["index"]]
        elif e["family"] == "ks_dmma" and e["dtype"] == "c64":
            assert (e["mr"] // 8, e["nr"] // 8) in gen.KSZ_TILES
        elif e["family"] in ("ks_fma", "ks1_fma"):
            # K-streamed entries: only those the install-time register check
            # (tools/ks_regs.py -> gen/ks_unroll.json) accepted
            assert 1 <= e["mr"] <= 8 and 1 <= e["nr"] <= 8
            assert gen.ks_unroll(e["dtype"], e["trans"], e["mr"], e["nr"]) > 0
        else:
            assert e["family"] in ("dmma", "ks_dmma")
            assert e["dtype"] == "f64" and e["mr"] % 8 == 0 and e["nr"] % 8 == 0
    # every (mr, nr) <= 4 x 4 exists for every dtype/trans: any M, N has an exact cover
    for dt in ("f32", "f64"):
        for tr in TRANS:
            for mr, nr in itertools.product(range(1, 5), repeat=2):
                assert ("fma", dt, tr, mr, nr) in CATSET


def test_not_small_and_invalid():
    with pytest.raises(iaat.IaatError):
        plan(0, "NN", 81, 81, 81)
    with pytest.raises(iaat.IaatError):
        plan(0, "TN", 33, 33, 33)


def _forced(**kw):
    import os
    keys = ("IAAT_FORCE_FAMILY", "IAAT_FORCE_TILE", "IAAT_FORCE_P", "IAAT_FORCE_CTAS", "IAAT_FORCE_ORDER")
    for k in keys:
        os.environ.pop(k, None)
    for k, v in kw.items():
        os.environ["IAAT_FORCE_" + k.upper()] = str(v)


def ks_cover(p, M, N):
    """Exact cover under the K-streamed element maps: MN-major dims tile
    contiguously, K-major dims interleave (row = base + t + tiles*i)."""
    tr = p["trans"]
    ak, bk = tr[0] == "T", tr[1] == "N"
    cover = np.zeros((M, N), dtype=np.int32)
    for c in p["classes"]:
        tm, tn = c["tm"], c["tiles"] // c["tm"]
        for ti, tj in itertools.product(range(tm), range(tn)):
            rows = [c["row_base"] + (ti + tm * i if ak else ti * c["mr"] + i) for i in range(c["mr"])]
            cols = [c["col_base"] + (tj + tn * j if bk else tj * c["nr"] + j) for j in range(c["nr"])]
            for r in rows:
                for q in cols:
                    cover[r, q] += 1
    return np.all(cover == 1)


@pytest.mark.parametrize("fam", [2, 6])
def test_forced_k_streamed_plans_are_valid(fam):
    """K-streamed plans (families 2 = KS/KS1, 6 = uniform-phase) over a grid
    of shapes: exact cover with their element maps, catalog membership,
    <= 16 resident warps per SM, smem within the opt-in limit, 1024-aligned
    stage regions, and the uniform-phase precondition."""
    try:
        for tr in TRANS:
            for (M, N, K) in ((64, 64, 64), (80, 72, 48), (36, 44, 52), (16, 24, 33), (48, 48, 48), (8, 40, 16)):
                if tr == "TN" and M * N * K > 32768:
                    continue
                for P in (1, 2, 3):
                    _forced(family=fam, p=P)
                    p = plan(0, tr, M, N, K, batch=5000)
                    if not p["family"].startswith("ks"):
                        continue  # not applicable: falls back to the slab planner
                    assert ks_cover(p, M, N), (tr, M, N, K, P, p["classes"])
                    fam_name = p["family"]
                    for c in p["classes"]:
                        assert (fam_name if fam_name != "ks_fma" else "ks_fma", "f32", tr, c["mr"], c["nr"]) in CATSET
                    assert p["ctas_per_sm"] * (p["compute_warps"] + 1) <= 16
                    assert p["smem"] * p["ctas_per_sm"] <= 228 * 1024
                    assert p["a_bytes"] % 1024 == 0 and p["b_bytes"] % 1024 == 0
                    assert p["block"] == 32 * (p["compute_warps"] + 1)
                    if fam_name == "ksu_fma":
                        c = p["classes"][0]
                        if tr[0] == "T":
                            assert c["tm"] % 8 == 0
                        if tr[1] == "N":
                            assert (c["tiles"] // c["tm"]) % 8 == 0
    finally:
        _forced()


def test_fp64_default_is_k_streamed_dmma(monkeypatch):
    """fp64 with M, N multiples of 8 and 16-byte aligned operands plans the
    K-streamed DMMA kernels by default (cost model, no install-time table);
    warps = P x warp tiles, one warp tile each; the MN-major pitch is
    4 (mod 16) doubles (conflict-free fragment rows)."""
    monkeypatch.setenv("IAAT_NO_TUNING", "1")
    for tr in ("NN", "NT", "TT"):
        for n in (16, 32, 48, 64, 80):
            p = plan(1, tr, n, n, n, batch=200000, beta0=True)
            assert p["family"] == "ks_dmma", (tr, n, p["family"])
            c = p["classes"][0]
            assert p["compute_warps"] == p["P"] * c["tiles"]
            assert (n // c["mr"]) * (n // c["nr"]) == c["tiles"]
            if tr[0] == "N":
                assert p["a_pitch"] % 16 == 4
            if tr[1] == "T":
                assert p["b_pitch"] % 16 == 4


def test_column_pair_eligibility():
    """Column-pair TMA boxes (planner.cpp plan_ksg, pairv): only packed operands
    with even extents whose ld's miss the 16-byte rule; everything else keeps
    its family (regular ksg boxes when the ld's are 16-byte multiples)."""
    for tr in ("NN", "NT", "TT"):
        p = plan(0, tr, 38, 38, 38)
        assert p["family"] == "ksg" and p["pairv"] == 1 and p["c_pitch"] == 38, p
        check_ksg_plan(p, tr, 38, 38)
        p = plan(0, tr, 40, 40, 40)
        assert p["family"] == "ksg" and p["pairv"] == 0, p
        # padded ld's (not packed), odd extents, 4-byte-aligned bases: not the pair view
        for kw in ({"pad": 2}, {"align": 4}, {"align": 8}):
            q = plan(0, tr, 38, 38, 38, **kw)
            assert q["family"] != "ksg", (kw, q)
        for (M, N, K) in ((37, 38, 38), (38, 37, 38), (39, 39, 39)):
            q = plan(0, tr, M, N, K)
            assert q["family"] != "ksg", (M, N, K, q)
    # an odd K leaves an MN-major operand with an odd column count (NN: A, NT: A and B, TT: B)
    assert plan(0, "NN", 38, 38, 37)["family"] != "ksg"
    # M a 16-byte multiple but N = ldb-rows not (NT: B is N x K): pair view for all three operands
    p = plan(0, "NT", 40, 38, 36)
    assert p["family"] == "ksg" and p["pairv"] == 1 and p["c_pitch"] == 40, p
