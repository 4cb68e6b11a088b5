"""GPU parity of the ksg family (csrc/iaat_ksg.cuh: lane-grid register
tiles, warp groups, C through shared memory, TMA zero fill past M / N).

Every catalog entry is forced (IAAT_FORCE_FAMILY=7, IAAT_FORCE_ORDER=entry)
on exact and zero-filled (Mv > M, Nv > N) tilings, ragged K chunks (K % KC,
K % 4 != 0), a ragged last unit (batch % P), beta != 0 and beta == 0 with a
NaN-filled C, and compared element-wise with the oracle
and bitwise with the slab family (one k-ascending FFMA chain per element and
the same fused epilogue in every family, reading A7).
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from tests.gpu_utils import Case, sample_ids

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

F32 = np.float32


def _force(**kw):
    for k in ("IAAT_FORCE_FAMILY", "IAAT_FORCE_TILE", "IAAT_FORCE_P", "IAAT_FORCE_CTAS", "IAAT_FORCE_ORDER",
              "IAAT_FORCE_S", "IAAT_FORCE_CSMEM"):
        os.environ.pop(k, None)
    for k, v in kw.items():
        os.environ["IAAT_FORCE_" + k.upper()] = str(v)


def _entries():
    from paper_2208_09822_b200 import iaat
    return [e for e in iaat.iaat_catalog_describe() if e["family"] == "ksg"]


def bits_equal(a, b):
    return torch.equal(a.view(torch.int32), b.view(torch.int32))


SHAPES = [(40, 40, 40), (48, 48, 48), (56, 56, 56), (64, 64, 64), (72, 72, 72), (80, 80, 80),
          (76, 76, 76), (44, 52, 37), (61, 70, 50), (80, 36, 100), (33, 64, 130), (68, 76, 98)]


def _plan(c, beta):
    from paper_2208_09822_b200 import iaat
    return iaat.iaat_plan_describe(0, c.tA, c.tB, c.M, c.N, c.K, c.lda, c.sA, c.ldb, c.sB, c.ldc, c.sC,
                                   c.batch, beta == 0)


@pytest.mark.parametrize("tr", ["NN", "NT", "TT"])
def test_ksg_every_entry_parity_and_bitwise_vs_slab(tr):
    ents = [e for e in _entries() if e["trans"] == tr]
    assert ents, "no ksg entries for %s" % tr
    ran = 0
    try:
        for e in ents:
            for (M, N, K) in SHAPES:
                for beta in (0.5, 0.0):
                    _force(family=7, order=e["index"])
                    c = Case(F32, tr[0], tr[1], M, N, K, 301, 31, 1.5, beta, ld_multiple=4)
                    p = _plan(c, beta)
                    if p.get("family") != "ksg" or p.get("entry") != e["index"]:
                        continue
                    A, B, C = c.views()
                    if beta == 0:
                        C.fill_(float("nan"))  # C is write-only at beta == 0 (reading A3)
                    c.run()
                    torch.cuda.synchronize()
                    c.check(sample_ids(c.batch, 48, 24))
                    got = C.clone()
                    _force(family=0)
                    c2 = Case(F32, tr[0], tr[1], M, N, K, 301, 31, 1.5, beta, ld_multiple=4)
                    if beta == 0:
                        c2.views()[2].fill_(float("nan"))
                    c2.run()
                    torch.cuda.synchronize()
                    assert bits_equal(got, c2.views()[2]), (tr, e, M, N, K, beta)
                    ran += 1
    finally:
        _force()
    assert ran >= 2 * len(ents), ran


PV_SHAPES = [(38, 38, 38), (42, 50, 46), (78, 78, 78), (66, 70, 62), (58, 34, 74), (40, 40, 38), (36, 38, 40),
             (74, 46, 18), (50, 50, 50)]


@pytest.mark.parametrize("tr", ["NN", "NT", "TT"])
def test_ksg_column_pair_boxes_every_entry(tr):
    """Column-pair TMA boxes (csrc/iaat_ksg.cuh PV; planner.cpp plan_ksg): packed
    operands with even ld's that are not multiples of 4 (8-byte column
    pitches).  Every catalog entry forced on such shapes -- ragged K chunks, a
    ragged last unit, rows past M that alias the next column (predicated
    stores), beta == 0 with a NaN-filled C -- against the oracle and bitwise
    against the slab family (the whole packed C: every neighbour intact)."""
    ents = [e for e in _entries() if e["trans"] == tr]
    ran = 0
    try:
        for e in ents:
            for i, (M, N, K) in enumerate(PV_SHAPES):
                beta = 0.0 if i % 3 == 1 else 0.5
                spad = 8 if i % 4 == 3 else 0  # gapped problem strides (16-byte multiples)
                _force(family=7, order=e["index"])
                c = Case(F32, tr[0], tr[1], M, N, K, 301, 37, 1.5, beta, spad=spad)
                p = _plan(c, beta)
                if p.get("family") != "ksg" or p.get("entry") != e["index"] or not p.get("pairv"):
                    continue
                A, B, C = c.views()
                if beta == 0:
                    C.fill_(float("nan"))
                c.run()
                torch.cuda.synchronize()
                c.check(sample_ids(c.batch, 48, 24))
                got = c.C.clone()
                _force(family=0)
                c2 = Case(F32, tr[0], tr[1], M, N, K, 301, 37, 1.5, beta, spad=spad)
                if beta == 0:
                    c2.views()[2].fill_(float("nan"))
                c2.run()
                torch.cuda.synchronize()
                assert bits_equal(got, c2.C), (tr, e, M, N, K, beta)
                ran += 1
    finally:
        _force()
    assert ran >= 2 * len(ents), ran


def test_ksg_column_pair_default_plan_full_batch():
    """n = 2 mod 4 squares at the held-out sweep's batch (256 MiB of operands):
    the default plan is a ksg column-pair plan; first / last / random problems
    against the oracle."""
    for n in (38, 58, 78):
        for tr in ("NN", "NT", "TT"):
            batch = (256 << 20) // (3 * n * n * 4)
            c = Case(F32, tr[0], tr[1], n, n, n, batch, 11, 1.5, 0.5)
            p = _plan(c, 0.5)
            assert p["family"] == "ksg" and p["pairv"] == 1, p
            c.run()
            torch.cuda.synchronize()
            c.check(sample_ids(c.batch, 128, 256))


def test_ksg_padding_and_gaps_untouched():
    """ld > rows and gapped problem strides: the TMA store writes exactly
    the M x N elements of every problem (NaN sentinels in the gaps stay)."""
    try:
        for tr in ("NN", "NT", "TT"):
            _force(family=7)
            c = Case(F32, tr[0], tr[1], 76, 72, 64, 257, 5, 1.0, 0.25, pad=4, spad=12)
            p = _plan(c, 0.25)
            assert p["family"] == "ksg", p
            c.run()
            torch.cuda.synchronize()
            c.check(sample_ids(c.batch, 32, 16))
            C = c.views()[2].cpu().numpy()
            mask = np.ones(C.shape, bool)
            for b in range(c.batch):
                for j in range(c.N):
                    o = b * c.sC + j * c.ldc
                    mask[o:o + c.M] = False
            assert np.isnan(C[mask]).all(), tr
    finally:
        _force()


def test_ksg_default_plans_and_small_batches():
    """The default plan picks ksg for the large config-2 shapes; batches
    smaller than one unit per group, and batch 1, are exact too."""
    for tr in ("NN", "NT", "TT"):
        for batch in (1, 3, 150, 1201):
            c = Case(F32, tr[0], tr[1], 80, 80, 80, batch, 8, -0.75, 1.25)
            c.run()
            torch.cuda.synchronize()
            c.check()


TN_SHAPES = [(31, 31, 31), (17, 17, 17), (23, 29, 19), (32, 32, 2), (13, 9, 21), (27, 27, 27), (5, 31, 29)]
SLAB_SHAPES = [(37, 67, 79), (67, 67, 17), (79, 79, 79), (33, 61, 47), (38, 38, 38), (61, 53, 31), (47, 79, 5)]


@pytest.mark.parametrize("tr", ["NN", "NT", "TT", "TN"])
def test_ksgs_every_entry_odd_shapes_parity_and_bitwise_vs_slab(tr):
    """ksgs (slab-staged lane grids): odd ld's, element-misaligned bases and
    padded ld's (the TMA rules exclude all of them), every entry forced
    (IAAT_FORCE_FAMILY=8), against the oracle and bitwise against the slab
    family; beta == 0 with a NaN-filled C."""
    ents = [e for e in iaat_entries("ksgs") if e["trans"] == tr]
    assert ents
    ran = 0
    try:
        for e in ents:
            for i, (M, N, K) in enumerate(SLAB_SHAPES if tr != "TN" else TN_SHAPES):
                beta = 0.0 if i % 3 == 2 else 0.5
                extra = [{}, {"pad": 1}, {"elem_offset": 1}][i % 3]
                _force(family=8, order=e["index"])
                c = Case(F32, tr[0], tr[1], M, N, K, 211, 41, -0.75, beta, **extra)
                p = _plan(c, beta)
                if p.get("family") != "ksgs" or p.get("entry") != e["index"]:
                    continue
                A, B, C = c.views()
                if beta == 0:
                    C.fill_(float("nan"))
                c.run()
                torch.cuda.synchronize()
                c.check(sample_ids(c.batch, 48, 24))
                got = c.C.clone()
                _force(family=0)
                c2 = Case(F32, tr[0], tr[1], M, N, K, 211, 41, -0.75, beta, **extra)
                if beta == 0:
                    c2.views()[2].fill_(float("nan"))
                c2.run()
                torch.cuda.synchronize()
                assert bits_equal(got, c2.C), (tr, e, M, N, K, beta, extra)
                ran += 1
    finally:
        _force()
    assert ran >= len(ents), ran


def iaat_entries(fam):
    from paper_2208_09822_b200 import iaat
    return [e for e in iaat.iaat_catalog_describe() if e["family"] == fam]


@pytest.mark.parametrize("tr", ["NN", "NT", "TT", "TN"])
def test_ksgs_shared_ring_wraps(tr):
    """ksgs's one ring of S stages shared by G groups (csrc/iaat_ksg.cuh
    SmemS): a batch large enough that every CTA runs more than 2S units, so
    every stage is refilled and both mbarrier phases recur; every entry
    forced, the smallest and the largest S the planner allows (IAAT_FORCE_S),
    sampled against the oracle, bitwise against the slab family; C through
    the stage (span store by the producer) and through global (CSMEM=0)."""
    ents = [e for e in iaat_entries("ksgs") if e["trans"] == tr]
    shapes = [(37, 67, 79), (31, 37, 37), (79, 31, 53)] if tr != "TN" else [(31, 31, 31), (17, 23, 19)]
    ran = 0
    try:
        for e in ents:
            for (M, N, K) in shapes:
                _force(family=8, order=e["index"])
                probe = Case(F32, tr[0], tr[1], M, N, K, 1, 7, 1.0, 1.0)
                p = _plan(probe, 1.0)
                if p.get("family") != "ksgs" or p.get("entry") != e["index"]:
                    continue
                G, S = e["g"], p["S"]
                for s, cs in sorted({(min(S, G + 1), 1), (S, 1), (S, 0)}):
                    batch = 148 * G * p["P"] * (2 * s + 1) + 5  # + a ragged last unit
                    _force(family=8, order=e["index"], s=s, **({} if cs else {"csmem": 0}))
                    c = Case(F32, tr[0], tr[1], M, N, K, batch, 43, 1.25, -0.5)
                    p2 = _plan(c, -0.5)
                    assert p2.get("entry") == e["index"] and p2["S"] <= s, p2
                    assert (p2["c_bytes"] > 0) == (cs == 1 and e["mr"] * e["nr"] < 100), p2
                    c.run()
                    torch.cuda.synchronize()
                    c.check(sample_ids(c.batch, 64, 32))
                    got = c.C.clone()
                    _force(family=0)
                    c2 = Case(F32, tr[0], tr[1], M, N, K, batch, 43, 1.25, -0.5)
                    c2.run()
                    torch.cuda.synchronize()
                    assert bits_equal(got, c2.C), (tr, e, M, N, K, s)
                    ran += 1
                break
    finally:
        _force()
    assert ran >= len(ents), ran
