#!/usr/bin/env python3
"""Probe the K-streamed (TMA) family on the GPU: parity of forced plans
against the oracle and timing of a knob grid, per shape.

    python tools/ks_probe.py f32 NN 80 [f32 TT 64 ...]
"""
import itertools
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2208_09822_b200.tune import Bench, set_knobs  # noqa: E402


def parity(dtype, tr, n, knobs, batch=700):
    from gpu_utils import Case
    set_knobs(**knobs)
    try:
        c = Case(np.float32 if dtype == "f32" else np.float64, tr[0], tr[1], n, n, n, batch, 5, 1.5, 0.5)
        c.run()
        import torch
        torch.cuda.synchronize()
        err, _, _ = c.check()
        c2 = Case(np.float32 if dtype == "f32" else np.float64, tr[0], tr[1], n, n, n, 301, 6, -1.0, 0.0)
        c2.run()
        err2, _, _ = c2.check()
        return max(err, err2)
    finally:
        set_knobs()


def main():
    args = sys.argv[1:]
    shapes = [(args[i], args[i + 1], int(args[i + 2])) for i in range(0, len(args), 3)]
    for dtype, tr, n in shapes:
        elt = 4 if dtype == "f32" else 8
        batch = (256 << 20) // (3 * n * n * elt)
        b = Bench(dtype, tr, n, n, n, batch, 1.5, 0.5)
        res = []
        set_knobs()
        base = b.time_us()
        print("%s %s n=%d batch=%d: default plan %.1f us  plan=%s" % (dtype, tr, n, b.batch, base,
                                                                    b.plan()["family"]), flush=True)
        if dtype == "f64":
            tiles = ["%dx%d" % (8 * a, 8 * b) for a in range(1, 6) for b in range(1, 6) if a * b <= 16]
            grid = [dict(family=3, tile=t, p=P, ctas=c) for t in tiles for P in (1, 2, 3, 4) for c in (1, 2, 3)]
        else:
            tiles = ["4x8", "8x4", "4x4", "6x8", "8x6", "5x8", "8x5", "4x6", "6x4"]
            grid = [dict(family=2, tile=t, order=o, p=P, ctas=c)
                    for t, o, P, c in itertools.product(tiles, (0, 1, 5, 9), (1, 2, 3, 4), (1, 2, 3, 4))]
        if os.environ.get("KS_PROBE_FAM") == "6":
            grid = [dict(family=6, tile=t, order=o, p=P, ctas=c)
                    for t, o, P, c in itertools.product(["8x8", "8x6", "6x8", "8x4", "4x8"], (0, 1, 3, 5, 9, 17),
                                                        (1, 2, 3, 4, 6), (1, 2, 3, 4))]
        for kw in grid:
            set_knobs(**kw)
            try:
                p = b.plan()
                if p["status"] != 0 or not p["family"].startswith("ks"):
                    continue
                key = (kw["family"], kw["tile"], p["classes"][0]["bm"], p["classes"][0]["colfast"], p["P"], p["ctas_per_sm"])
                if any(r[2] == key for r in res):
                    continue
                us = b.time_us()
            except Exception as e:  # noqa: BLE001
                print("  fail", kw, e)
                continue
            finally:
                set_knobs()
            res.append((us, kw, key, p["S"], p["compute_warps"]))
        res.sort(key=lambda r: r[0])
        byts = (3 + 1) * n * n * elt * b.batch
        for us, kw, key, S, W in res[:8]:
            print("  %.1f us  %.0f GB/s  %.0f GFLOP/s  %s S=%d W=%d" % (us, byts / us / 1e3,
                                                                       2.0 * n ** 3 * b.batch / us / 1e3, kw, S, W))
        b.free()
        for us, kw, key, S, W in res[:3]:
            err = parity(dtype, tr, n, kw)
            print("  parity %s: max rel err %.2e" % (kw, err), flush=True)


if __name__ == "__main__":
    main()
