"""the paper-faithful tiling mode (iaat_paper_tile; host only, no
GPU).  Pinned to the paper's own numbers (Fig. 2's 72K + 450 for 15 x 15,
PAPER.md:337; Alg. 2's fixed branches), to Table I
(tests/golden/table1_sgemm_nn.json), and to an independent
brute-force search over all strip compositions."""
from __future__ import annotations

import functools
import json
import os

import pytest

from paper_2208_09822_b200 import iaat

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table1_sgemm_nn.json")))
TABLE = {int(k): v for k, v in GOLD["blocks"].items()}


def blocks(plan):
    for s in plan["strips"]:
        for w, n in s["n"]:
            for _ in range(s["count"] * n):
                yield s["h"], w


def check_cover(plan, M, N):
    assert sum(s["h"] * s["count"] for s in plan["strips"]) == M
    for s in plan["strips"]:
        assert sum(w * n for w, n in s["n"]) == N
    for h, w in blocks(plan):
        assert h in TABLE and w in TABLE[h], (h, w)  # only Table I kernels
    # memops of PAPER.md:310 recomputed from the blocks
    assert plan["memops_k_coeff"] == sum(h + w for h, w in blocks(plan))
    assert plan["memops_const"] == 2 * M * N


def test_fig2_15x15_optimum_is_72k_plus_450():
    p = iaat.iaat_paper_tile(1, 15, 15)
    check_cover(p, 15, 15)
    assert p["memops_k_coeff"] == GOLD["fig2_15x15"]["k_coeff"]
    assert p["memops_const"] == GOLD["fig2_15x15"]["const"]


def test_alg2_literal_15x15_reading_a14():
    # DESIGN.md A14: a literal trace of Alg. 2 gives 8/4/3 strips, 75K + 450 (not Fig. 2's 72)
    p = iaat.iaat_paper_tile(0, 15, 15)
    check_cover(p, 15, 15)
    assert [s["h"] for s in p["strips"]] == [8, 4, 3]
    assert p["memops_k_coeff"] == 75


def test_alg2_fixed_branches():
    # M == 9 -> (4, 1), (3, 1), (2, 1)  (Alg. 2)
    p = iaat.iaat_paper_tile(0, 9, 40)
    assert [(s["h"], s["count"]) for s in p["strips"]] == [(4, 1), (3, 1), (2, 1)]
    # M == 12 -> one 12-high strip tiled with widths <= 6
    p = iaat.iaat_paper_tile(0, 12, 40)
    assert [(s["h"], s["count"]) for s in p["strips"]] == [(12, 1)]
    assert max(w for w, _ in p["strips"][0]["n"]) <= 6
    # 8 < M < 12 -> (8, 1), (M - 8, 1)
    p = iaat.iaat_paper_tile(0, 11, 40)
    assert [(s["h"], s["count"]) for s in p["strips"]] == [(8, 1), (3, 1)]
    # N <= 13 -> n_c = N, m_1 the largest m_c with a kernel of width N
    p = iaat.iaat_paper_tile(0, 40, 7)
    assert p["strips"][0]["h"] == 8 and p["strips"][0]["n"] == [[7, 1]] and p["strips"][0]["count"] == 5
    p = iaat.iaat_paper_tile(0, 40, 4)
    assert p["strips"][0]["h"] == 16 and p["strips"][0]["count"] == 2 and p["strips"][1]["h"] == 8


@functools.lru_cache(maxsize=None)
def brute(M, N):
    """Independent exhaustive minimum of sum(m_i + n_i) over row strips of
    Table I heights, each strip tiled in N by any Table I widths of its height
    (plain recursion, no shared code with the library)."""
    @functools.lru_cache(maxsize=None)
    def row(h, n):
        if n == 0:
            return 0
        return min(h + w + row(h, n - w) for w in TABLE[h] if w <= n)

    @functools.lru_cache(maxsize=None)
    def col(m):
        if m == 0:
            return 0
        return min(row(h, N) + col(m - h) for h in TABLE if h <= m)

    return col(M)


def test_optimum_matches_brute_force_and_bounds_literal():
    for M in range(1, 25):
        for N in range(1, 25):
            opt = iaat.iaat_paper_tile(1, M, N)
            lit = iaat.iaat_paper_tile(0, M, N)
            check_cover(opt, M, N)
            check_cover(lit, M, N)
            assert opt["memops_k_coeff"] == brute(M, N), (M, N)
            assert opt["memops_k_coeff"] <= lit["memops_k_coeff"], (M, N)


def test_covers_up_to_80():
    for M in range(1, 81, 7):
        for N in range(1, 81, 5):
            for mode in (0, 1):
                check_cover(iaat.iaat_paper_tile(mode, M, N), M, N)


def test_invalid():
    with pytest.raises(iaat.IaatError):
        iaat.iaat_paper_tile(2, 4, 4)
    with pytest.raises(iaat.IaatError):
        iaat.iaat_paper_tile(0, 0, 4)
