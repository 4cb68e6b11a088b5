#!/usr/bin/env python3
"""Does a plan's time depend on what ran before it?  Times one shape under
two knob sets, (1) called back to back (the tuner's setting) and (2) each
call preceded by a call of another shape (the bench's setting).

    python tools/context_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2208_09822_b200.tune import Bench, set_knobs  # noqa: E402


def timed(torch, fn_main, fn_other, reps, interleave):
    tot = 0.0
    for _ in range(reps):
        if interleave:
            fn_other()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn_main()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot * 1e3 / reps


def main():
    import torch
    cases = [("NT", 64, {}, dict(tile="4x8", p=3, csmem=1, order=0, ctas=1, s=2)),
             ("NN", 64, {}, dict(tile="4x8", p=2, csmem=1, order=17, ctas=1, s=2)),
             ("TT", 68, {}, dict(tile="4x8", p=2, csmem=1, order=0, ctas=1, s=3))]
    other = Bench("f32", "NN", 60, 60, 60, (256 << 20) // (12 * 3600), 1.5, 0.5)
    for tr, n, ka, kb in cases:
        b = Bench("f32", tr, n, n, n, (256 << 20) // (12 * n * n), 1.5, 0.5)
        for name, kw in (("table", ka), ("tuned", kb)):
            set_knobs(**kw)
            b.call()
            torch.cuda.synchronize()
            iso = timed(torch, b.call, other.call, 10, False)
            seq = timed(torch, b.call, other.call, 10, True)
            set_knobs()
            print("f32 %s %d %-6s %s: back-to-back %.1f us, after another shape %.1f us" % (tr, n, name, kw, iso, seq),
                  flush=True)
        b.free()


if __name__ == "__main__":
    main()
