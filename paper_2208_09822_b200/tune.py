"""Install-time tuning on a B200 (run once per machine type, result committed).

    python -m paper_2208_09822_b200.tune --config 2 [--config 3 ...] [--out .../tuning/b200.tsv]

The paper's install-time stage "automatically tunes kernels based on
features of the hardware" (Sec. I; Sec. III-A).
Here the hardware-dependent choices are the run-time planner's knobs: the
main micro-tile of the exact decomposition, problems per stage P, pipeline
stages S, CTAs per SM and the lane -> tile mapping.  For each input of a
workload this script times candidate plans through the public C ABI (forced
with the IAAT_FORCE_* knobs the planner understands), keeps the fastest, and
writes one line per input to tuning/b200.tsv, which libiaat.so reads at run
time (key: dtype, transposition, M, N, K, ld's, packed strides, beta == 0,
16-byte alignment).  Inputs not in the table fall back to the planner's cost
model.  Tuning only changes speed: every candidate computes the same
bitwise-identical result (one fixed-order FMA chain per element).
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
DEFAULT_OUT = os.path.join(PKG, "tuning", "b200.tsv")
KNOBS = ("IAAT_FORCE_TILE", "IAAT_FORCE_P", "IAAT_FORCE_S", "IAAT_FORCE_CTAS", "IAAT_FORCE_ORDER",
         "IAAT_FORCE_FAMILY", "IAAT_FORCE_CSMEM")
S3 = [1, 3, 5, 7, 11, 13, 17, 23, 31, 37, 47, 53, 61, 67, 79]


def config_shapes(cfg):
    """(dtype, trans, M, N, K, batch, alpha, beta) of BASELINE.json's configs."""
    out = []
    if cfg == 1:
        out.append(("f32", "NN", 16, 16, 16, 2000, 1.0, 0.0))
    elif cfg == 2:
        for n in range(4, 81, 4):
            for tr in ("NN", "NT", "TT"):
                out.append(("f32", tr, n, n, n, (256 << 20) // (12 * n * n), 1.5, 0.5))
    elif cfg == 3:
        triples = [(m, n, k) for m in S3 for n in S3 for k in S3 if m * n * k <= 512000]
        rng = np.random.default_rng(2)
        for i in rng.choice(len(triples), size=64, replace=False):
            m, n, k = triples[i]
            out.append(("f32", "NN", m, n, k, 100000, 1.0, 1.0))
    elif cfg == 4:
        for n in range(2, 33):
            out.append(("f32", "TN", n, n, n, 500000, -1.0, 0.25))
        out += [("f32", "TN", 32, 32, 2, 500000, -1.0, 0.25), ("f32", "TN", 2, 32, 32, 500000, -1.0, 0.25)]
    elif cfg == 5:
        for n in (8, 16, 32, 48, 64, 80):
            for tr in ("NN", "NT"):
                out.append(("f64", tr, n, n, n, 2_000_000, 1.0, 0.0))
    elif cfg == 6:  # complex fp32 sweep (bench.py --config 6)
        for n in range(4, 81, 4):
            for tr in ("NN", "NT", "TT"):
                out.append(("c32", tr, n, n, n, (256 << 20) // (24 * n * n), 1.5 - 0.5j, 0.5 + 0.25j))
    elif cfg == 7:  # complex fp64 sweep (bench.py --config 7)
        for n in (8, 16, 24, 32, 40, 48, 56, 64, 80):
            for tr in ("NN", "NT", "TT"):
                out.append(("c64", tr, n, n, n, (256 << 20) // (48 * n * n), 1.5 - 0.5j, 0.5 + 0.25j))
    elif cfg == 8:  # fp32 TN above 32^3 (bench.py --config 8; needs iaat_set_tn_limit)
        for n in range(36, 81, 4):
            out.append(("f32", "TN", n, n, n, (256 << 20) // (12 * n * n), 1.5, 0.5))
    elif cfg == 9:  # fp64 TN / TT (bench.py --config 9)
        for n in range(8, 81, 8):
            for tr in ("TN", "TT"):
                out.append(("f64", tr, n, n, n, (256 << 20) // (24 * n * n), 1.5, 0.5))
    return out


def set_knobs(**kw):
    for k in KNOBS:
        os.environ.pop(k, None)
    for k, v in kw.items():
        if v is not None:
            os.environ["IAAT_FORCE_" + k.upper()] = str(v)


class Bench:
    """One input of the workload, with NSETS independent operand sets used
    round-robin so that consecutive timed calls never find the previous
    call's operands in L2 (each set is >= 2x the 126 MB L2 or the full
    workload batch, whichever is smaller)."""
    NSETS = 3

    def __init__(self, dtype, tr, M, N, K, batch, alpha, beta, max_bytes=3 << 30):
        import torch
        import datagen
        self.torch = torch
        self.dt = {"f32": 0, "f64": 1, "c32": 2, "c64": 3}[dtype]
        elt = {"f32": 4, "f64": 8, "c32": 8, "c64": 16}[dtype]
        w = 2 if dtype in ("c32", "c64") else 1  # complex: interleaved (re, im) pairs
        self.tr, self.M, self.N, self.K, self.alpha, self.beta = tr, M, N, K, alpha, beta
        ra, ca = (M, K) if tr[0] == "N" else (K, M)
        rb, cb = (K, N) if tr[1] == "N" else (N, K)
        per = (ra * ca + rb * cb + M * N) * elt
        self.batch = int(min(batch, max(1, max_bytes // per)))
        self.ra, self.ca, self.rb, self.cb = ra, ca, rb, cb
        tdt = torch.float32 if dtype in ("f32", "c32") else torch.float64
        nsets = self.NSETS if self.batch * per < (1 << 30) else 1
        self.sets = []
        for i in range(nsets):
            A = torch.empty(w * self.batch * ra * ca, dtype=tdt, device="cuda")
            B = torch.empty(w * self.batch * rb * cb, dtype=tdt, device="cuda")
            C = torch.empty(w * self.batch * M * N, dtype=tdt, device="cuda")
            datagen.fill_device(A, 9 + i, 0, w * ra, ca, w * ra, w * ra * ca, self.batch)
            datagen.fill_device(B, 9 + i, 1, w * rb, cb, w * rb, w * rb * cb, self.batch)
            datagen.fill_device(C, 9 + i, 2, w * M, N, w * M, w * M * N, self.batch)
            self.sets.append((A, B, C))
        self.turn = 0

    def plan(self):
        from paper_2208_09822_b200 import iaat
        return iaat.iaat_plan_describe(self.dt, self.tr[0], self.tr[1], self.M, self.N, self.K, self.ra,
                                       self.ra * self.ca, self.rb, self.rb * self.cb, self.M, self.M * self.N,
                                       self.batch, self.beta == 0)

    def call(self):
        from paper_2208_09822_b200 import iaat
        A, B, C = self.sets[self.turn % len(self.sets)]
        self.turn += 1
        st = iaat.iaat_gemm_strided_batched(self.dt, self.tr[0], self.tr[1], self.M, self.N, self.K, self.alpha,
                                            A.data_ptr(), self.ra, self.ra * self.ca, B.data_ptr(),
                                            self.rb, self.rb * self.cb, self.beta, C.data_ptr(), self.M,
                                            self.M * self.N, self.batch,
                                            self.torch.cuda.current_stream().cuda_stream)
        if st != 0:
            raise RuntimeError("status %d" % st)

    def time_us(self, reps=6, warm=3):
        """Mean time of one call.  Each timed call is preceded by a call of
        another, small problem shape (the separator), as in bench.py's
        sequence of shapes: a kernel that follows itself overlaps its tail
        with the next launch of the same kernel, which a kernel following a
        different one (other smem carve-out) cannot -- back-to-back timing
        favoured plans that lose in the real sequence (tools/context_probe.py)."""
        torch = self.torch
        sep = separator()

        def sep_call():  # the separator runs its own (untuned, unforced) plan
            saved = {k: os.environ.pop(k) for k in KNOBS if k in os.environ}
            try:
                sep.call()
            finally:
                os.environ.update(saved)

        for _ in range(warm):
            sep_call()
            self.call()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for e0, e1 in ev:
            sep_call()
            e0.record()
            self.call()
            e1.record()
        torch.cuda.synchronize()
        return sum(e0.elapsed_time(e1) for e0, e1 in ev) * 1e3 / reps

    def free(self):
        del self.sets
        self.torch.cuda.empty_cache()


_SEP = []


def separator():
    """A small fixed call (fp32 NN 24^3, 16 MiB of operands) run between timed calls."""
    if not _SEP:
        saved = {k: os.environ.pop(k) for k in KNOBS if k in os.environ}
        try:
            _SEP.append(Bench("f32", "NN", 24, 24, 24, (16 << 20) // (12 * 24 * 24), 1.0, 0.5, max_bytes=64 << 20))
        finally:
            os.environ.update(saved)
    return _SEP[0]


def key_line(dt, tr, M, N, K, beta0):
    """The planner's tuning-table key for a packed strided call with 256 B
    aligned bases (csrc/planner.cpp make_plan): the 16-byte vector legality
    field must be the planner's own (every ld and problem stride a multiple
    of 16 bytes) or the entry never matches."""
    ra = M if tr[0] == "N" else K
    rb = K if tr[1] == "N" else N
    ca = K if tr[0] == "N" else M
    cb = N if tr[1] == "N" else K
    elt = (4, 8, 8, 16)[dt]
    al = lambda el: (el * elt) % 16 == 0  # noqa: E731
    vec = int(al(ra) and al(rb) and al(M) and al(ra * ca) and al(rb * cb) and al(M * N))
    return "%d %d %d %d %d %d %d %d %d %d %d %d" % (dt, tr[0] == "T", tr[1] == "T", M, N, K, ra, rb, M, 1,
                                                     int(beta0), vec)


def tile_options(M, N, wide=False):
    """First-strip tile sizes to try.  wide: also 3, 5, 6 (the exact-cover
    planner pairs them with a second strip), for the large fp32 shapes."""
    base = (2, 3, 4, 5, 6, 8) if wide else (2, 4, 8)
    ms = sorted({x for x in (1, 2, 3, 4, 5, 6, 7, 8) if x <= M and (x in base or x == M or M < 8)})
    ns = sorted({x for x in (1, 2, 3, 4, 5, 6, 7, 8) if x <= N and (x in base or x == N or N < 8)})
    return [(a, b) for a in ms for b in ns if not wide or a * b >= 12]


def tune_shape(sh, log):
    dtype, tr, M, N, K, batch, alpha, beta = sh
    elt = {"f32": 4, "f64": 8, "c32": 8, "c64": 16}[dtype]
    b = Bench(*sh)
    results = []  # (us, knobs dict)

    def trial(**kw):
        set_knobs(**kw)
        try:
            p = b.plan()
            if p["status"] != 0:
                return None
            if kw.get("family") in (2, 3, 6) and not p["family"].startswith("ks"):
                return None  # K-streamed plan not applicable: the planner fell back
            us = b.time_us()
        except Exception:
            return None
        finally:
            set_knobs()
        results.append((us, kw, p))
        return us

    auto = trial()
    per = (M * K + K * N + (0 if beta == 0 else M * N)) * elt
    Ps = sorted({max(1, int(kb * 1024) // per) for kb in (12, 24, 40, 64, 96)})
    for (mr, nr) in tile_options(M, N):
        for P in Ps:
            trial(tile="%dx%d" % (mr, nr), p=P)
    if dtype == "f64" and M % 8 == 0 and N % 8 == 0:
        for (wm, wn) in ((1, 1), (1, 2), (2, 1), (2, 2)):
            for P in Ps:
                trial(tile="%dx%d" % (8 * wm, 8 * wn), p=P, family=1)
    if dtype in ("f64", "c64") and M % 8 == 0 and N % 8 == 0:  # K-streamed DMMA warp tiles (ZGEMM too)
        for a in range(1, 6):
            for bb in range(1, 6):
                if a * bb <= 16 and 8 * a <= M and 8 * bb <= N:
                    for P in (1, 2, 3, 4):
                        for ctas in (1, 2, 3):
                            trial(family=3, tile="%dx%d" % (8 * a, 8 * bb), p=P, ctas=ctas)
    if max(M, N, K) >= 20:  # K-streamed TMA family (csrc/iaat_ks.cuh)
        ks_tiles = [t for t in ("4x8", "8x4", "4x4", "6x8", "8x6", "5x8", "8x5", "4x6", "6x4", "2x8", "8x2")
                    if int(t.split("x")[0]) <= M and int(t.split("x")[1]) <= N]
        for tile in ks_tiles:
            for order in (0, 1, 5, 9):
                for P in (1, 2, 3, 4):
                    for ctas in (1, 2, 3, 4):
                        trial(family=2, tile=tile, order=order, p=P, ctas=ctas)
    if dtype == "f32" and tr != "TN" and max(M, N, K) >= 24:  # uniform-phase K-streamed big tiles
        for tile in ("8x8", "8x6", "6x8", "8x4", "4x8"):
            for order in (0, 5, 9, 17):
                for P in (1, 2, 3, 4):
                    for ctas in (1, 2, 3, 4):
                        trial(family=6, tile=tile, order=order, p=P, ctas=ctas)
    if dtype == "f32" and min(M, N) >= 48:  # wider first-strip grid for the FFMA-bound sizes
        for (mr, nr) in tile_options(M, N, wide=True):
            if (mr, nr) in tile_options(M, N):
                continue
            for P in (1, 2, 3):
                for csm in ((0, 1) if beta != 0 else (None,)):
                    trial(tile="%dx%d" % (mr, nr), p=P, csmem=csm)
    if beta != 0:  # C_in from global (L2-prefetched) or staged in smem, both explicitly
        per_ab = (M * K + K * N) * elt
        for (mr, nr) in tile_options(M, N):
            for P in sorted({max(1, int(kb * 1024) // per_ab) for kb in (24, 48, 96)}):
                trial(tile="%dx%d" % (mr, nr), p=P, csmem=0)
            for P in (1, 2, 3):
                trial(tile="%dx%d" % (mr, nr), p=P, csmem=1)
    results.sort(key=lambda x: x[0])
    top = [r for r in results if r[1].get("family") not in (2, 3, 6)][:4]
    for us, kw, p in top:
        for order in (0, 1, 3, 5, 9, 17):
            for ctas in (1, 2, 3, 4):
                for s in (0, 2, 3):
                    for csm in ((None, 0, 1) if beta != 0 else (None,)):
                        kk = dict(kw)
                        kk.update(order=order, ctas=ctas)
                        if s:
                            kk["s"] = s
                        if csm is not None:
                            kk["csmem"] = csm
                        trial(**kk)
    # one timing per trial is noisy: re-time the leaders (and the automatic
    # plan) with more repetitions and keep the best of those
    results.sort(key=lambda x: x[0])
    seen, lead = set(), []
    for us, kw, p in results:
        key = tuple(sorted(kw.items()))
        if key not in seen:
            seen.add(key)
            lead.append(kw)
        if len(lead) == 5:
            break
    if {} not in lead:
        lead.append({})
    first_pass = results
    results = []
    for kw in lead:
        set_knobs(**kw)
        try:
            p = b.plan()
            if p["status"] == 0:
                results.append((min(b.time_us(reps=12), b.time_us(reps=12)), kw, p))
        except Exception:
            pass
        finally:
            set_knobs()
    if not results:
        results = first_pass
    results.sort(key=lambda x: x[0])
    auto = next((us for us, kw, p in results if kw == {}), auto)
    best_us, best_kw, best_p = results[0]
    b.free()
    if auto is not None and auto <= best_us * 1.01:
        best_kw, best_us = {}, auto
    byts = (M * K + K * N + M * N * (1 if beta == 0 else 2)) * elt * b.batch
    fl = (8.0 if dtype in ("c32", "c64") else 2.0) * M * N * K * b.batch
    log("%s %s %dx%dx%d batch=%d auto=%.1fus best=%.1fus (%.0f GB/s, %.0f GFLOP/s) knobs=%s" % (
        dtype, tr, M, N, K, b.batch, auto or -1, best_us, byts / best_us / 1e3, fl / best_us / 1e3, best_kw))
    return best_kw, best_p


def line_to_knobs(v):
    """Inverse of knobs_to_line: a table entry's fields as IAAT_FORCE_* knobs."""
    mr, nr, P, S, ctas, order, fam, csm = (int(x) for x in v.split()[:8])
    kw = {}
    if mr:
        kw["tile"] = "%dx%d" % (mr, nr)
    for k, x, none in (("p", P, 0), ("s", S, 0), ("ctas", ctas, 0), ("order", order, -1), ("family", fam, -1),
                       ("csmem", csm, -1)):
        if x != none:
            kw[k] = x
    return kw


def tune_ksg(sh, current, log):
    """ksg / ksgs families (csrc/iaat_ksg.cuh) against the current plan of one
    input: every applicable catalog entry (forced), each at its planner-chosen ring
    depth and one stage fewer, plus the current table entry (or the cost
    model's plan); the leaders are re-timed and the fastest is kept."""
    from paper_2208_09822_b200 import iaat
    dtype, tr, M, N, K, batch, alpha, beta = sh
    b = Bench(*sh)
    cands = [current or {}]
    for e in iaat.iaat_catalog_describe():
        if e["family"] not in ("ksg", "ksgs") or e["trans"] != tr:
            continue
        fam = 7 if e["family"] == "ksg" else 8
        set_knobs(family=fam, order=e["index"])
        try:
            p = b.plan()
        finally:
            set_knobs()
        if p.get("family") != e["family"] or p.get("entry") != e["index"]:
            continue
        cands.append({"family": fam, "order": e["index"]})
        if p["S"] > 1:
            cands.append({"family": fam, "order": e["index"], "s": p["S"] - 1})
        if fam == 8:  # ksgs: C through global instead of through the stage
            cands.append({"family": fam, "order": e["index"], "csmem": 0})
    res = []
    for kw in cands:
        set_knobs(**kw)
        try:
            p = b.plan()
            if p["status"] == 0:
                res.append((b.time_us(), kw, p))
        except Exception as ex:  # a candidate that cannot run is skipped, not fatal
            log("  candidate %s failed: %s" % (kw, ex))
        finally:
            set_knobs()
    res.sort(key=lambda x: x[0])
    final = []
    for us, kw, p in res[:4] + [r for r in res if r[1] == cands[0]][:1]:
        set_knobs(**kw)
        try:
            final.append((min(b.time_us(reps=12), b.time_us(reps=12)), kw, p))
        except Exception as ex:
            log("  candidate %s failed: %s" % (kw, ex))
        finally:
            set_knobs()
    final.sort(key=lambda x: x[0])
    cur = next((us for us, kw, p in final if kw == cands[0]), float("inf"))
    best_us, best_kw, best_p = final[0]
    b.free()
    if best_kw != cands[0] and best_us > cur * 0.99:
        best_kw, best_us, best_p = cands[0], cur, None
    byts = (M * K + K * N + M * N * (1 if beta == 0 else 2)) * 4 * b.batch
    log("ksg %s %dx%dx%d batch=%d current=%.1fus best=%.1fus (%.0f GB/s) knobs=%s" % (
        tr, M, N, K, b.batch, cur, best_us, byts / best_us / 1e3, best_kw))
    return best_kw, best_p


def knobs_to_line(kw, p):
    """Knobs of the winning plan as the planner's table fields."""
    mr, nr = (int(x) for x in kw["tile"].split("x")) if "tile" in kw else (0, 0)
    return "%d %d %d %d %d %d %d %d" % (mr, nr, kw.get("p", 0), kw.get("s", 0), kw.get("ctas", 0),
                                        kw.get("order", -1), kw.get("family", -1), kw.get("csmem", -1))


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, action="append", default=[])
    ap.add_argument("--out", default=DEFAULT_OUT)
    ap.add_argument("--log", default=None)
    ap.add_argument("--min-n", type=int, default=0, help="only inputs with max(M,N,K) >= this")
    ap.add_argument("--max-n", type=int, default=1 << 30)
    ap.add_argument("--ksg", action="store_true", help="only compare the ksg family against the current entries")
    a = ap.parse_args(argv)
    sys.path.insert(0, ROOT)
    os.environ["IAAT_NO_TUNING"] = "1"  # tune against the cost model, not an older table
    if set(a.config) & {8, 9}:
        from paper_2208_09822_b200 import iaat
        iaat.iaat_set_tn_limit(512000)  # TN above the paper's 32^3
    existing = {}
    if os.path.exists(a.out):
        for ln in open(a.out):
            if ln.startswith("#") or ":" not in ln:
                continue
            k, v = ln.split(":", 1)
            existing[k.strip()] = v.strip()
    logf = open(a.log, "a") if a.log else None

    def log(s):
        print(s, flush=True)
        if logf:
            logf.write(s + "\n")
            logf.flush()

    t0 = time.time()
    for cfg in a.config or [2]:
        for sh in config_shapes(cfg):
            if not a.min_n <= max(sh[2:5]) <= a.max_n:
                continue
            dtype, tr, M, N, K, batch, alpha, beta = sh
            key = key_line({"f32": 0, "f64": 1, "c32": 2, "c64": 3}[dtype], tr, M, N, K, beta == 0)
            if a.ksg:
                if dtype != "f32" or min(M, N) < (13 if tr == "TN" else 11):
                    continue
                kw, p = tune_ksg(sh, line_to_knobs(existing[key]) if key in existing else {}, log)
            else:
                kw, p = tune_shape(sh, log)
            if kw:
                existing[key] = knobs_to_line(kw, p)
            else:
                existing.pop(key, None)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        f.write("# install-time tuning table for libiaat.so on B200 (written by paper_2208_09822_b200/tune.py)\n")
        f.write("# dtype tA tB M N K lda ldb ldc packed beta0 vec : mr nr P S ctas order family csmem\n")
        for k in sorted(existing):
            f.write("%s : %s\n" % (k, existing[k]))
    log("tuned %d entries in %.0fs -> %s" % (len(existing), time.time() - t0, a.out))


if __name__ == "__main__":
    main()
