#!/usr/bin/env python3
"""Wider knob grid than tune.py for a few config-2 shapes (slab family):
tile x P x CTAs/SM x stages x C_in staging, timed through the C ABI.

    python tools/slab_probe.py TT 68 [NN 76 ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2208_09822_b200.tune import Bench, set_knobs  # noqa: E402


def main():
    a = sys.argv[1:]
    for tr, n in zip(a[0::2], a[1::2]):
        n = int(n)
        b = Bench("f32", tr, n, n, n, (256 << 20) // (12 * n * n), 1.5, 0.5)
        base = b.time_us()
        res = []
        for tile in ("4x8", "8x4", "4x4", "4x6", "6x4", "2x8", "8x2", "4x5", "5x4", "3x8", "8x3"):
            for P in (1, 2, 3):
                for ctas in (1, 2, 3):
                    for s in (2, 3):
                        for csmem in (0, 1):
                            set_knobs(tile=tile, p=P, ctas=ctas, s=s, csmem=csmem)
                            try:
                                pl = b.plan()
                                if pl["status"] != 0 or pl["family"] != "fma" or pl["ctas_per_sm"] != ctas:
                                    continue
                                us = b.time_us()
                            except Exception:
                                continue
                            finally:
                                set_knobs()
                            res.append((us, dict(tile=tile, p=P, ctas=ctas, s=s, csmem=csmem)))
        res.sort(key=lambda x: x[0])
        print("f32 %s %d: tuned %.1f us; best %s" % (tr, n, base, ["%.1f %s" % r for r in res[:4]]), flush=True)
        b.free()


if __name__ == "__main__":
    main()
