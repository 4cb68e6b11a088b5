#!/usr/bin/env python3
"""Probe the K-streamed family's LDGSTS mode (misaligned, odd-ld inputs) on
the GPU: tuned plan vs forced K-streamed plans over tiles x P x CTAs, with a parity check of the best forced plan.

    python tools/ldgsts_probe.py 37 67 79 [67 67 17 ...]   (fp32 NN, alpha=1, beta=1, batch 100000)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2208_09822_b200.tune import Bench, set_knobs  # noqa: E402


def main():
    a = [int(x) for x in sys.argv[1:]]
    for M, N, K in zip(a[0::3], a[1::3], a[2::3]):
        b = Bench("f32", "NN", M, N, K, 100000, 1.0, 1.0)
        base = b.time_us()
        best = (1e30, None)
        for tile in ("4x4", "4x8", "8x4", "2x8", "8x2", "4x6", "6x4", "2x4", "4x2"):
            mr, nr = map(int, tile.split("x"))
            if mr > M or nr > N:
                continue
            for P in (1, 2, 3):
                for ctas in (1, 2, 3):
                    set_knobs(family=2, tile=tile, p=P, ctas=ctas)
                    try:
                        pl = b.plan()
                        if pl["status"] != 0 or not pl["family"].startswith("ks"):
                            continue
                        us = b.time_us()
                    except Exception:
                        continue
                    finally:
                        set_knobs()
                    if us < best[0]:
                        best = (us, dict(tile=tile, p=P, ctas=ctas))
        print("f32 NN %dx%dx%d: tuned %.1f us, best LDGSTS KS %.1f us %s" % (M, N, K, base, best[0], best[1]),
              flush=True)
        b.free()
        if best[1]:
            from gpu_utils import Case
            set_knobs(family=2, **best[1])
            try:
                c = Case(np.float32, "N", "N", M, N, K, 997, 5, 1.5, 0.5)
                c.run()
                err, _, _ = c.check()
                print("   parity max rel err %.2e" % err, flush=True)
            finally:
                set_knobs()


if __name__ == "__main__":
    main()
