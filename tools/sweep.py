#!/usr/bin/env python3
"""Planner tuning sweep: time one shape under forced plans (IAAT_FORCE_*).

    python tools/sweep.py f32 NN 64 [--tiles 8x8,4x8] [--P 1,2,3] [--S 2,3,4]
Prints one line per (tile, P, S): us, GB/s, GFLOP/s, plan summary.
"""
import argparse
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("dtype")
    ap.add_argument("trans")
    ap.add_argument("n", type=int)
    ap.add_argument("--tiles", default="")
    ap.add_argument("--P", default="")
    ap.add_argument("--S", default="")
    ap.add_argument("--beta", type=float, default=0.5)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--family", default="")
    ap.add_argument("--stage-kb", default="", help="derive P from target stage KB (A+B+C_in)")
    a = ap.parse_args()
    import torch
    import datagen
    from paper_2208_09822_b200 import iaat
    n = a.n
    elt = 4 if a.dtype == "f32" else 8
    batch = a.batch or (256 << 20) // (3 * n * n * elt)
    tdt = torch.float32 if elt == 4 else torch.float64
    A = torch.empty(batch * n * n, dtype=tdt, device="cuda")
    B = torch.empty_like(A)
    C = torch.empty_like(A)
    for i, t in enumerate((A, B, C)):
        datagen.fill_device(t, 1, i, n, n, n, n * n, batch)
    dt = 0 if elt == 4 else 1
    tiles = a.tiles.split(",") if a.tiles else [""]
    Ps = [int(x) for x in a.P.split(",")] if a.P else [0]
    if a.stage_kb:
        per = (3 if a.beta else 2) * n * n * elt
        Ps = sorted(set(max(1, int(float(x) * 1024) // per) for x in a.stage_kb.split(",")))
    Ss = [int(x) for x in a.S.split(",")] if a.S else [0]
    byts = (3 + (1 if a.beta else 0)) * n * n * elt * batch
    for tile, P, S in itertools.product(tiles, Ps, Ss):
        for k in ("IAAT_FORCE_TILE", "IAAT_FORCE_P", "IAAT_FORCE_S", "IAAT_FORCE_FAMILY"):
            os.environ.pop(k, None)
        if tile:
            os.environ["IAAT_FORCE_TILE"] = tile
        if P:
            os.environ["IAAT_FORCE_P"] = str(P)
        if S:
            os.environ["IAAT_FORCE_S"] = str(S)
        if a.family:
            os.environ["IAAT_FORCE_FAMILY"] = a.family
        try:
            plan = iaat.iaat_plan_describe(dt, a.trans[0], a.trans[1], n, n, n, n, n * n, n, n * n, n, n * n,
                                           batch, a.beta == 0)
        except Exception as e:
            print(tile, P, S, "plan failed", e)
            continue
        if plan["status"] != 0:
            print(tile, P, S, "no plan")
            continue
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        try:
            for r in range(3):
                iaat.gemm_strided_batched(a.trans[0], a.trans[1], n, n, n, 1.5, A, n, n * n, B, n, n * n, a.beta, C,
                                          n, n * n, batch)
            ev[0].record()
            for r in range(5):
                iaat.gemm_strided_batched(a.trans[0], a.trans[1], n, n, n, 1.5, A, n, n * n, B, n, n * n, a.beta, C,
                                          n, n * n, batch)
            ev[1].record()
            torch.cuda.synchronize()
        except Exception as e:
            print(tile, P, S, "run failed", e)
            continue
        us = ev[0].elapsed_time(ev[1]) * 1e3 / 5
        cls = ",".join("%dx%d:%d-%d" % (c["mr"], c["nr"], c["warp_begin"], c["warp_end"]) for c in plan["classes"])
        print("%s %s n=%d tile=%s P=%d S=%d W=%d smem=%d c_smem=%d | %.1f us %.0f GB/s %.0f GFLOP/s | %s" % (
            a.dtype, a.trans, n, tile or "auto", plan["P"], plan["S"], plan["compute_warps"], plan["smem"],
            plan["c_in_smem"], us, byts / us / 1e3, 2.0 * n ** 3 * batch / us / 1e3, cls), flush=True)


if __name__ == "__main__":
    main()
