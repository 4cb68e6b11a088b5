#!/usr/bin/env python3
"""Held-out sweep: is the run-time planner input-aware
without per-shape tuning?  Times, through the public C ABI, fp32 shapes that
are NOT in the install-time tuning table -- M = N = K = n with n = 2 (mod 4)
(38 ... 78; TMA-illegal odd-granule ld's are part of the test) and 64 random
(M, N, K) with M != N != K -- for NN / NT / TT, each with the planner's cost
model alone (IAAT_NO_TUNING=1; the table cannot match these keys anyway), and
the tuned config-2 neighbours n - 2 and n + 2 for comparison.  Batch: 256 MiB
of operands per shape (config-2 recipe), alpha = 1.5, beta = 0.5.

    python tools/heldout.py --out profiles/r02/heldout_r02.json
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def frac(M, N, K, batch, us, hbm=6550.1, ffma=74.4):
    byts = (M * K + K * N + 2 * M * N) * 4.0 * batch
    t = max(byts / (hbm * 1e9), 2.0 * M * N * K * batch / (ffma * 1e12))
    return t / (us * 1e-6)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    from paper_2208_09822_b200.tune import Bench
    rng = np.random.default_rng(7)
    shapes = [(n, n, n) for n in range(38, 80, 4)]
    while len(shapes) < 12 + 64:
        M, N, K = (int(x) for x in rng.integers(20, 81, size=3))
        if len({M, N, K}) == 3 and M * N * K <= 512000:
            shapes.append((M, N, K))
    out = []
    for (M, N, K) in shapes:
        for tr in ("NN", "NT", "TT"):
            batch = (256 << 20) // ((M * K + K * N + M * N) * 4)
            rec = {"M": M, "N": N, "K": K, "trans": tr, "batch": batch}
            os.environ["IAAT_NO_TUNING"] = "1"
            b = Bench("f32", tr, M, N, K, batch, 1.5, 0.5)
            rec["family"] = b.plan()["family"]
            us = min(b.time_us(reps=8), b.time_us(reps=8))
            rec["us"] = round(us, 2)
            rec["frac"] = round(frac(M, N, K, b.batch, us), 4)
            b.free()
            if M == N == K:
                os.environ.pop("IAAT_NO_TUNING", None)
                nb = []
                for n2 in (M - 2, M + 2):
                    bb = Bench("f32", tr, n2, n2, n2, (256 << 20) // (12 * n2 * n2), 1.5, 0.5)
                    u2 = min(bb.time_us(reps=8), bb.time_us(reps=8))
                    nb.append(round(frac(n2, n2, n2, bb.batch, u2), 4))
                    bb.free()
                rec["tuned_neighbours_frac"] = nb
            out.append(rec)
            print(json.dumps(rec), flush=True)
    sq = [r for r in out if "tuned_neighbours_frac" in r]
    summary = {
        "square_heldout_mean_frac": float(np.mean([r["frac"] for r in sq])),
        "square_tuned_neighbours_mean_frac": float(np.mean([np.mean(r["tuned_neighbours_frac"]) for r in sq])),
        "random_mean_frac": float(np.mean([r["frac"] for r in out if r not in sq])),
        "within_10pct_of_neighbours": int(sum(r["frac"] >= 0.9 * np.mean(r["tuned_neighbours_frac"]) for r in sq)),
        "square_count": len(sq),
    }
    with open(a.out, "w") as f:
        json.dump({"summary": summary, "records": out}, f, indent=1)
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
