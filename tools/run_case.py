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
    elt = {"f32": 4, "f64": 8, "c32": 8, "c64": 16}[a.dtype]
    w = 2 if a.dtype in ("c32", "c64") else 1  # complex: interleaved (re, im) real view
    if a.batch == 0:
        a.batch = (256 << 20) // ((a.M * a.K + a.K * a.N + a.M * a.N) * elt)
    ra, ca = (a.M, a.K) if a.trans[0] == "N" else (a.K, a.M)
    rb, cb = (a.K, a.N) if a.trans[1] == "N" else (a.N, a.K)
    tdt = torch.float32 if a.dtype in ("f32", "c32") else torch.float64
    A = torch.empty(w * a.batch * ra * ca, dtype=tdt, device="cuda")
    B = torch.empty(w * a.batch * rb * cb, dtype=tdt, device="cuda")
    C = torch.empty(w * a.batch * a.M * a.N, dtype=tdt, device="cuda")
    datagen.fill_device(A, 1, 0, w * ra, ca, w * ra, w * ra * ca, a.batch)
    datagen.fill_device(B, 1, 1, w * rb, cb, w * rb, w * rb * cb, a.batch)
    datagen.fill_device(C, 1, 2, w * a.M, a.N, w * a.M, w * a.M * a.N, a.batch)
    dt = {"f32": 0, "f64": 1, "c32": 2, "c64": 3}[a.dtype]
    if a.plan:
        print(iaat.iaat_plan_describe(dt, a.trans[0], a.trans[1], a.M, a.N, a.K, ra, ra * ca, rb, rb * cb,
                                      a.M, a.M * a.N, a.batch, a.beta == 0))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for r in range(a.reps):
        if r == a.reps - 1:
            ev[0].record()
        st = iaat.iaat_gemm_strided_batched(dt, a.trans[0], a.trans[1], a.M, a.N, a.K, a.alpha, A.data_ptr(), ra,
                                            ra * ca, B.data_ptr(), rb, rb * cb, a.beta, C.data_ptr(), a.M, a.M * a.N,
                                            a.batch, torch.cuda.current_stream().cuda_stream)
        assert st == 0, iaat.iaat_status_string(st)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    byts = (a.M * a.K + a.K * a.N + a.M * a.N * (2 if a.beta else 1)) * elt * a.batch
    fl = (8.0 if w == 2 else 2.0) * a.M * a.N * a.K * a.batch
    print("%s %s %dx%dx%d batch=%d: %.1f us, %.1f GFLOP/s, %.1f GB/s" % (
        a.dtype, a.trans, a.M, a.N, a.K, a.batch, ms * 1e3, fl / ms / 1e6, byts / ms / 1e6))


if __name__ == "__main__":
    main()
