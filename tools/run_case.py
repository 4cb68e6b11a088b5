#!/usr/bin/env python3
"""Run one (dtype, trans, M, N, K, batch) batched call a few times -- the
unit the ncu captures in profiles/ are taken on.

    python tools/run_case.py f32 NN 32 32 32 [batch] [--reps 4] [--alpha 1.5 --beta 0.5]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("dtype")
    ap.add_argument("trans")
    ap.add_argument("M", type=int)
    ap.add_argument("N", type=int)
    ap.add_argument("K", type=int)
    ap.add_argument("batch", type=int, nargs="?", default=0)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--alpha", type=float, default=1.5)
    ap.add_argument("--beta", type=float, default=0.5)
    ap.add_argument("--plan", action="store_true")
    a = ap.parse_args()
    import torch
    import datagen
    from paper_2208_09822_b200 import iaat
    elt = 4 if a.dtype == "f32" else 8
    if a.batch == 0:
        a.batch = (256 << 20) // ((a.M * a.K + a.K * a.N + a.M * a.N) * elt)
    ra, ca = (a.M, a.K) if a.trans[0] == "N" else (a.K, a.M)
    rb, cb = (a.K, a.N) if a.trans[1] == "N" else (a.N, a.K)
    tdt = torch.float32 if elt == 4 else torch.float64
    A = torch.empty(a.batch * ra * ca, dtype=tdt, device="cuda")
    B = torch.empty(a.batch * rb * cb, dtype=tdt, device="cuda")
    C = torch.empty(a.batch * a.M * a.N, dtype=tdt, device="cuda")
    datagen.fill_device(A, 1, 0, ra, ca, ra, ra * ca, a.batch)
    datagen.fill_device(B, 1, 1, rb, cb, rb, rb * cb, a.batch)
    datagen.fill_device(C, 1, 2, a.M, a.N, a.M, a.M * a.N, a.batch)
    dt = 0 if elt == 4 else 1
    if a.plan:
        print(iaat.iaat_plan_describe(dt, a.trans[0], a.trans[1], a.M, a.N, a.K, ra, ra * ca, rb, rb * cb,
                                      a.M, a.M * a.N, a.batch, a.beta == 0))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for r in range(a.reps):
        if r == a.reps - 1:
            ev[0].record()
        iaat.gemm_strided_batched(a.trans[0], a.trans[1], a.M, a.N, a.K, a.alpha, A, ra, ra * ca, B, rb, rb * cb,
                                  a.beta, C, a.M, a.M * a.N, a.batch)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    byts = (a.M * a.K + a.K * a.N + a.M * a.N * (2 if a.beta else 1)) * elt * a.batch
    print("%s %s %dx%dx%d batch=%d: %.1f us, %.1f GFLOP/s, %.1f GB/s" % (
        a.dtype, a.trans, a.M, a.N, a.K, a.batch, ms * 1e3, 2.0 * a.M * a.N * a.K * a.batch / ms / 1e6,
        byts / ms / 1e6))


if __name__ == "__main__":
    main()
