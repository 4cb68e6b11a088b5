#!/usr/bin/env python3
"""Benchmark: batched small GEMM GFLOP/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 1..5]

Default workload (BASELINE.json configs[1], "config2"): fp32 square sweep
M=N=K in {4,8,...,80} x trans in {NN,NT,TT}, each shape with
batch = floor(256 MiB / ((MK+KN+MN)*4 B)) independent column-major problems,
alpha=1.5, beta=0.5, inputs uniform[-1,1) from the seeded counter generator
(datagen/, seed 1).  One STEP = the 60 library calls of the sweep.
Inputs are resident in HBM before the timed region; every call touches its own
256 MiB (> 126 MB L2), so consecutive calls cannot hit in L2.

value     = whole-job GFLOP/s = sum over ranks of 2*M*N*K*batch per step / time
e2e       = the same metric through the C ABI with HOST (pinned) buffers: H2D of
            A, B, C and D2H of C inside the timed region
roofline  = the dominant launch (largest share of the step): algorithmic bytes
            (MK+KN+2MN)*4*batch (or 2MNK*batch flops if FFMA-bound) / its
            average CUDA-event duration, vs MEASURED_PEAKS.json
cpu_baseline = the CPU oracle (oracle/ref_gemm.c, OpenMP, all host cores) on
            a bounded sample of the same step (rank 0, N=1 only)

Multi-GPU (torchrun, one process per GPU): every rank runs the full sweep on
its own problems (weak scaling, no collective on the data path); barrier +
synchronize around the timed region, time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "batched small GEMM GFLOP/s per B200 and % of roofline vs M=N=K, 1/2/4/8 GPUs"
FFMA_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.4, derived
DMMA_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12    # 37.2, derived


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def roofline_of(s, cnt, t, pk):
    """Roofline object of one launch (shape s, cnt problems, t seconds):
    HBM-bound -> algorithmic GB/s vs the measured copy bandwidth; otherwise
    flops vs the derived FFMA (fp32, "alu") or DMMA (fp64, "tensor") peak."""
    hbm_time = s.alg_bytes(cnt) / (pk["hbm_gbs"] * 1e9)
    fp32 = s.dtype in ("f32", "c32")
    cmp_peak = FFMA_PEAK_TFLOPS if fp32 else DMMA_PEAK_TFLOPS
    if hbm_time >= s.flops(cnt) / (cmp_peak * 1e12):
        roof = {"bound": "hbm", "achieved": round(s.alg_bytes(cnt) / t / 1e9, 1), "peak": pk["hbm_gbs"],
                "unit": "GB/s", "frac": round(s.alg_bytes(cnt) / t / 1e9 / pk["hbm_gbs"], 4),
                "peak_source": pk["source"]}
    else:
        roof = {"bound": "alu" if fp32 else "tensor", "achieved": round(s.flops(cnt) / t / 1e12, 2),
                "peak": round(cmp_peak, 1), "unit": "TFLOP/s",
                "frac": round(s.flops(cnt) / t / 1e12 / cmp_peak, 4),
                "peak_source": ("derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz (DESIGN.md)" if fp32 else
                                "derived: 148 SM x 64 FP64 FMA/clk (DMMA) x 2 x 1.965 GHz (DESIGN.md)")}
    roof["traffic"] = load_traffic(s.name(), cnt)
    return roof


# ---------------------------------------------------------------- workloads
class Shape:
    def __init__(self, dtype, tr, M, N, K, batch, alpha, beta, seed):
        self.dtype, self.tr, self.M, self.N, self.K = dtype, tr, M, N, K
        self.batch, self.alpha, self.beta, self.seed = batch, alpha, beta, seed

    @property
    def elt(self):
        return {"f32": 4, "f64": 8, "c32": 8, "c64": 16}[self.dtype]

    @property
    def cplx(self):
        return self.dtype in ("c32", "c64")

    @property
    def dt_index(self):
        return {"f32": 0, "f64": 1, "c32": 2, "c64": 3}[self.dtype]

    def stored(self):
        ra, ca = (self.M, self.K) if self.tr[0] == "N" else (self.K, self.M)
        rb, cb = (self.K, self.N) if self.tr[1] == "N" else (self.N, self.K)
        return ra, ca, rb, cb

    def flops(self, batch=None):
        # Eq. 1 (real) / Eq. 2 (complex: 8 flops per complex multiply-add)
        return (8.0 if self.cplx else 2.0) * self.M * self.N * self.K * (self.batch if batch is None else batch)

    def alg_bytes(self, batch=None):
        b = self.batch if batch is None else batch
        cbytes = self.M * self.N * (2 if self.beta != 0 else 1)
        return float(self.M * self.K + self.K * self.N + cbytes) * self.elt * b

    def formula_bytes(self, batch=None):
        b = self.batch if batch is None else batch
        return float(self.M * self.K + self.K * self.N + 2 * self.M * self.N) * self.elt * b

    def name(self):
        return "%s_%s_%dx%dx%d" % (self.dtype, self.tr, self.M, self.N, self.K)


def workload(cfg):
    S = []
    if cfg == 1:
        S.append(Shape("f32", "NN", 16, 16, 16, 2000, 1.0, 0.0, 0))
        desc = "config1: fp32 NN M=N=K=16 batch=2000 alpha=1 beta=0 (latency-bound, L2-resident)"
    elif cfg == 2:
        for n in range(4, 81, 4):
            b = (256 * 1024 * 1024) // (3 * n * n * 4)
            for tr in ("NN", "NT", "TT"):
                S.append(Shape("f32", tr, n, n, n, b, 1.5, 0.5, 1))
        desc = ("config2: fp32 square sweep M=N=K in {4,8,...,80} x {NN,NT,TT}, "
                "batch=floor(256MiB/(3n^2*4B)), alpha=1.5, beta=0.5, seed 1")
    elif cfg == 3:
        from tests.gpu_utils import config3_shapes
        for (m, n, k) in config3_shapes():
            S.append(Shape("f32", "NN", m, n, k, 100000, 1.0, 1.0, 2))
        desc = "config3: fp32 NN, 64 irregular (M,N,K) from {1,3,...,79}^3, batch 100000 each, alpha=1, beta=1"
    elif cfg == 4:
        from tests.gpu_utils import config4_shapes
        for (m, n, k) in config4_shapes():
            S.append(Shape("f32", "TN", m, n, k, 500000, -1.0, 0.25, 3))
        desc = "config4: fp32 TN, M=N=K in 2..32 + (32,32,2), (2,32,32), batch 500000, alpha=-1, beta=0.25"
    elif cfg == 5:
        for n in (8, 16, 32, 48, 64, 80):
            for tr in ("NN", "NT"):
                S.append(Shape("f64", tr, n, n, n, 2_000_000, 1.0, 0.0, 4))
        desc = ("config5: fp64 NN/NT M=N=K in {8,16,32,48,64,80}, global batch 2e6 sharded across the GPUs by "
                "contiguous ranges (strong scaling), chunked to fit HBM, alpha=1, beta=0")
    elif cfg == 6:  # SURVEY f1 (not a BASELINE config): complex fp32, config-2 shape of sweep
        for n in range(4, 81, 4):
            b = (256 * 1024 * 1024) // (3 * n * n * 8)
            for tr in ("NN", "NT", "TT"):
                S.append(Shape("c32", tr, n, n, n, b, 1.5 - 0.5j, 0.5 + 0.25j, 1))
        desc = ("cgemm sweep (SURVEY f1): complex fp32 M=N=K in {4,...,80} x {NN,NT,TT}, batch=floor(256MiB/(3n^2*8B)), "
                "alpha=1.5-0.5i, beta=0.5+0.25i, seed 1; GFLOP/s by Eq. 2 (8MNK)")
    elif cfg == 7:  # complex fp64
        for n in (8, 16, 24, 32, 40, 48, 56, 64, 80):
            b = (256 * 1024 * 1024) // (3 * n * n * 16)
            for tr in ("NN", "NT", "TT"):
                S.append(Shape("c64", tr, n, n, n, b, 1.5 - 0.5j, 0.5 + 0.25j, 1))
        desc = ("zgemm sweep (SURVEY f1): complex fp64 M=N=K in {8,16,24,32,40,48,56,64,80} x {NN,NT,TT}, batch=floor(256MiB/(3n^2*16B)), "
                "alpha=1.5-0.5i, beta=0.5+0.25i, seed 1; GFLOP/s by Eq. 2 (8MNK)")
    elif cfg == 8:  # fp32 TN above the paper's 32^3 bound (iaat_set_tn_limit)
        for n in range(36, 81, 4):
            b = (256 * 1024 * 1024) // (3 * n * n * 4)
            S.append(Shape("f32", "TN", n, n, n, b, 1.5, 0.5, 1))
        desc = ("fp32 TN above 32^3 (SURVEY f2, iaat_set_tn_limit(80^3)): M=N=K in {36,...,80}, "
                "batch=floor(256MiB/(3n^2*4B)), alpha=1.5, beta=0.5, seed 1")
    elif cfg == 9:  # fp64 TN / TT
        for n in range(8, 81, 8):
            b = (256 * 1024 * 1024) // (3 * n * n * 8)
            for tr in ("TN", "TT"):
                S.append(Shape("f64", tr, n, n, n, b, 1.5, 0.5, 1))
        desc = ("fp64 TN/TT (SURVEY f2; TN above 32^3 via iaat_set_tn_limit(80^3)): M=N=K in {8,...,80}, "
                "batch=floor(256MiB/(3n^2*8B)), alpha=1.5, beta=0.5, seed 1")
    elif cfg == 10:  # held-out sweep: n = 2 (mod 4), no tuning-table entries
        for n in range(38, 80, 4):
            b = (256 * 1024 * 1024) // (3 * n * n * 4)
            for tr in ("NN", "NT", "TT"):
                S.append(Shape("f32", tr, n, n, n, b, 1.5, 0.5, 1))
        desc = ("held-out fp32 squares M=N=K in {38,42,...,78} x {NN,NT,TT} (8-byte column pitches: ksg column-pair TMA "
                "boxes, cost-model plans only), batch=floor(256MiB/(3n^2*4B)), alpha=1.5, beta=0.5, seed 1")
    else:
        raise SystemExit("unknown config %r" % cfg)
    return S, desc


def plan_chunks(shapes, cfg, rank, world, hbm_cap):
    """The calls one rank makes per step: (shape, first GLOBAL problem id,
    count).  Config 5 is strong scaling (BASELINE.json: a fixed batch of
    2,000,000 sharded across the GPUs by contiguous ranges): rank r owns
    dist.shard_range(batch, r, world) and splits it into chunks that fit 60 %
    of HBM.  Every other config is weak scaling: each rank runs the whole
    workload on its own problems [r*batch, (r+1)*batch).  Inputs are
    generated from the global ids, so a problem's data -- and its result --
    do not depend on the split."""
    from paper_2208_09822_b200.dist import shard_range
    chunks = []
    for s in shapes:
        if cfg == 5:
            lo, hi = shard_range(s.batch, rank, world)
            ra, ca, rb, cb = s.stored()
            per = (ra * ca + rb * cb + s.M * s.N) * s.elt
            cnt = max(1, min(hi - lo, int(0.60 * hbm_cap) // per))
            for c0 in range(lo, hi, cnt):
                chunks.append((s, c0, min(cnt, hi - c0)))
        else:
            chunks.append((s, rank * s.batch, s.batch))
    return chunks


# ---------------------------------------------------------------- clocks
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import datagen
    from paper_2208_09822_b200 import iaat

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    shapes, desc = workload(args.config)
    if any(s.tr == "TN" and s.M * s.N * s.K > 32768 for s in shapes):
        assert iaat.iaat_set_tn_limit(512000) == 0  # TN above the paper's 32^3
    stream = torch.cuda.current_stream()
    tdt = {"f32": torch.float32, "f64": torch.float64, "c32": torch.float32, "c64": torch.float64}

    # --- allocate + fill (outside the timed region); one buffer set per (dtype, M,N,K)
    hbm_cap = torch.cuda.get_device_properties(dev).total_memory
    bufs = {}
    chunks = plan_chunks(shapes, args.config, rank, world, hbm_cap)  # (shape, first global id, count)
    for s, lo, cnt in chunks:
        key = (s.dtype, s.M, s.N, s.K, s.tr, cnt)
        if key in bufs:
            continue
        if args.config == 5:
            bufs.clear()
            torch.cuda.empty_cache()
        ra, ca, rb, cb = s.stored()
        w = 2 if s.cplx else 1  # complex: interleaved (re, im) = a real (2*rows) x cols matrix
        A = torch.empty(w * cnt * ra * ca, dtype=tdt[s.dtype], device=dev)
        B = torch.empty(w * cnt * rb * cb, dtype=tdt[s.dtype], device=dev)
        C = torch.empty(w * cnt * s.M * s.N, dtype=tdt[s.dtype], device=dev)
        first = lo  # global problem ids: ranks own disjoint problems
        datagen.fill_device(A, s.seed, datagen.MAT_A, w * ra, ca, w * ra, w * ra * ca, cnt, first)
        datagen.fill_device(B, s.seed, datagen.MAT_B, w * rb, cb, w * rb, w * rb * cb, cnt, first)
        datagen.fill_device(C, s.seed, datagen.MAT_C, w * s.M, s.N, w * s.M, w * s.M * s.N, cnt, first)
        bufs[key] = (A, B, C)
        if args.config == 5:
            break  # config 5 re-fills per chunk inside the step loop (generation untimed, see below)
    A = B = C = None  # only bufs holds the operand sets (config 5 frees them chunk by chunk)
    torch.cuda.synchronize()

    def call(s, lo, cnt, strm=None):
        strm = stream if strm is None else strm
        ra, ca, rb, cb = s.stored()
        A, B, C = bufs[(s.dtype, s.M, s.N, s.K, s.tr, cnt)]
        st = iaat.iaat_gemm_strided_batched(s.dt_index, s.tr[0], s.tr[1], s.M, s.N, s.K,
                                            s.alpha, A.data_ptr(), ra, ra * ca, B.data_ptr(), rb, rb * cb,
                                            s.beta, C.data_ptr(), s.M, s.M * s.N, cnt, strm.cuda_stream)
        if st != 0:
            raise RuntimeError("iaat call failed: %s (%s)" % (iaat.iaat_status_string(st), s.name()))

    if args.config == 5:
        return run_chunked_config5(args, rank, world, local_rank, shapes, desc, chunks, bufs, call)
    if args.grouped:
        return run_grouped(args, rank, world, local_rank, shapes, desc, chunks, bufs, stream)

    def step(evs=None):
        for i, (s, lo, cnt) in enumerate(chunks):
            if evs is not None:
                evs[i][0].record(stream)
            call(s, lo, cnt)
            if evs is not None:
                evs[i][1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in chunks] for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local_rank)
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    n_launch0 = iaat.iaat_launch_count()
    # the timed region: K steps of back-to-back calls, events only at its
    # two ends (an event between two calls would stand between the kernels
    # in the stream and cost the programmatic-dependent-launch overlap)
    t0.record(stream)
    for k in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    n_launch = iaat.iaat_launch_count() - n_launch0
    clk = clocks.stop()
    barrier(world)
    ms_total = t0.elapsed_time(t1)
    ms_total = allreduce_max(ms_total, world)
    # per-call breakdown (roofline of the dominant launch, per-shape
    # fractions): a second, instrumented pass of K steps with an event pair
    # around every call -- not part of the timed value
    for k in range(args.steps):
        step(evs[k])
    torch.cuda.synchronize()
    per_call_ms = np.zeros(len(chunks))
    for k in range(args.steps):
        for i, (a, b) in enumerate(evs[k]):
            per_call_ms[i] += a.elapsed_time(b)
    per_call_ms /= args.steps

    flops_step = sum(s.flops(cnt) for s, lo, cnt in chunks)
    ms_step = ms_total / args.steps
    value = flops_step * world / (ms_step * 1e-3) / 1e9

    # per-shape breakdown + dominant launch roofline
    pk = peaks()
    shapes_out = []
    dom = int(np.argmax(per_call_ms))
    for i, (s, lo, cnt) in enumerate(chunks):
        t = per_call_ms[i] * 1e-3
        gf = s.flops(cnt) / t / 1e9
        t_roof = max(s.flops(cnt) / (FFMA_PEAK_TFLOPS * 1e12 if s.dtype in ("f32", "c32") else DMMA_PEAK_TFLOPS * 1e12),
                     s.alg_bytes(cnt) / (pk["hbm_gbs"] * 1e9))
        shapes_out.append({"shape": s.name(), "batch": cnt, "us": round(t * 1e6, 2), "gflops": round(gf, 1),
                           "hbm_gbs": round(s.alg_bytes(cnt) / t / 1e9, 1),
                           "frac_roofline": round(t_roof / t, 4)})
    s, lo, cnt = chunks[dom]
    tdom = per_call_ms[dom] * 1e-3
    roof = roofline_of(s, cnt, tdom, pk)
    roof["kernel"] = s.name()
    roof["share_of_step"] = round(per_call_ms[dom] / per_call_ms.sum(), 4)
    roof["bytes_per_launch"] = s.alg_bytes(cnt)
    roof["flops_per_launch"] = s.flops(cnt)

    # --- e2e through the C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, chunks, bufs, call, stream, world)

    line = {"metric": METRIC, "value": round(value, 1), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": shapes[0].dtype, "data": "synthetic",
            "config": {"workload": desc, "calls_per_step": len(chunks),
                       "l2": "inputs larger than L2: every call streams its own 256 MiB operand set "
                             "(126 MB L2), no flush kernel needed" if args.config in (2, 10) else
                             "as workload states", "parallelism": "dp%d (batch shards, no collective)" % world,
                       "timing": "K steps back to back, CUDA events at the two ends only; per-shape times "
                                 "and the roofline launch from a second pass with an event pair per call"},
            "roofline": roof, "gpu_launches": int(n_launch), "clocks": clk, "e2e": e2e,
            "shapes": shapes_out}
    if args.config == 1:
        line["hot_graph"] = run_graph_hot(chunks, call, stream)
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = run_cpu_baseline(shapes, args)
    return line


def run_graph_hot(chunks, call, stream, reps=100):
    """Config 1 is launch/latency-bound: one 16^3 x 2000 call is
    ~3 us of GPU work behind ~15 us of host submission.  Reported beside the
    per-call number, labelled: the same call captured 100 times back to back
    in a CUDA graph and replayed (operands L2-resident: 8 MB), device time per
    call.  Not the headline value."""
    import torch
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        for s, lo, cnt in chunks:
            call(s, lo, cnt, torch.cuda.current_stream())  # warm the plan cache on this stream
        with torch.cuda.graph(g, stream=side):
            for _ in range(reps):
                for s, lo, cnt in chunks:
                    call(s, lo, cnt, torch.cuda.current_stream())
    stream.wait_stream(side)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    fl = sum(s.flops(cnt) for s, lo, cnt in chunks)
    return {"us_per_call": round(us, 3), "gflops": round(fl / us / 1e3, 1), "calls": reps,
            "label": "hot: CUDA-graph replay of %d back-to-back calls, L2-resident operands" % reps}


def run_grouped(args, rank, world, local_rank, shapes, desc, chunks, bufs, stream):
    """the whole workload (e.g. config 3's 64 shapes) as ONE
    grouped call per step (iaat_gemm_grouped_strided: one plan per size
    class, groups enqueued back to back by the library)."""
    import torch
    from paper_2208_09822_b200 import iaat
    groups = []
    for s, lo, cnt in chunks:
        ra, ca, rb, cb = s.stored()
        A, B, C = bufs[(s.dtype, s.M, s.N, s.K, s.tr, cnt)]
        groups.append(dict(transA=s.tr[0], transB=s.tr[1], M=s.M, N=s.N, K=s.K, alpha=s.alpha, A=A.data_ptr(),
                           lda=ra, strideA=ra * ca, B=B.data_ptr(), ldb=rb, strideB=rb * cb, beta=s.beta,
                           C=C.data_ptr(), ldc=s.M, strideC=s.M * s.N, batch=cnt))
    dt = shapes[0].dt_index

    def step():
        st = iaat.iaat_gemm_grouped_strided(dt, groups, stream.cuda_stream)
        if st != 0:
            raise RuntimeError("grouped call failed: %s" % iaat.iaat_status_string(st))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local_rank)
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    n0 = iaat.iaat_launch_count()
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    n_launch = iaat.iaat_launch_count() - n0
    clk = clocks.stop()
    ms = allreduce_max(t0.elapsed_time(t1), world) / args.steps
    flops = sum(s.flops(cnt) for s, lo, cnt in chunks)
    byts = sum(s.alg_bytes(cnt) for s, lo, cnt in chunks)
    pk = peaks()
    return {"metric": METRIC, "value": round(flops * world / (ms * 1e-3) / 1e9, 1), "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": shapes[0].dtype,
            "data": "synthetic",
            "config": {"workload": desc + " -- as ONE grouped call per step (SURVEY f4)", "groups": len(groups)},
            "roofline": {"bound": "hbm", "achieved": round(byts / (ms * 1e-3) / 1e9, 1), "peak": pk["hbm_gbs"],
                         "unit": "GB/s", "frac": round(byts / (ms * 1e-3) / 1e9 / pk["hbm_gbs"], 4),
                         "traffic": None, "kernel": "whole grouped call (all %d groups)" % len(groups)},
            "gpu_launches": int(n_launch), "clocks": clk}


def run_chunked_config5(args, rank, world, local_rank, shapes, desc, chunks, bufs, call):
    """Config 5 (fp64, up to 307 GB of operands per shape): chunks that fit
    HBM; per chunk the inputs are generated (untimed) and the call timed with
    CUDA events; GEMM time is summed."""
    import torch
    import datagen
    from paper_2208_09822_b200 import iaat
    tdt = torch.float64
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream()
    res = {}
    n_launch = 0
    clocks = ClockSampler(local_rank)
    clocks.start()
    A = B = C = None
    for s, lo, cnt in chunks:
        key = (s.dtype, s.M, s.N, s.K, s.tr, cnt)
        if key not in bufs:
            A = B = C = None  # drop every reference before freeing
            bufs.clear()
            torch.cuda.empty_cache()
            ra, ca, rb, cb = s.stored()
            bufs[key] = (torch.empty(cnt * ra * ca, dtype=tdt, device=dev),
                         torch.empty(cnt * rb * cb, dtype=tdt, device=dev),
                         torch.empty(cnt * s.M * s.N, dtype=tdt, device=dev))
        A, B, C = bufs[key]
        ra, ca, rb, cb = s.stored()
        first = lo  # this rank's shard of the global batch (plan_chunks)
        datagen.fill_device(A, s.seed, datagen.MAT_A, ra, ca, ra, ra * ca, cnt, first)
        datagen.fill_device(B, s.seed, datagen.MAT_B, rb, cb, rb, rb * cb, cnt, first)
        for _ in range(args.warmup):
            call(s, lo, cnt)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n0 = iaat.iaat_launch_count()
        e0.record(stream)
        for _ in range(args.steps):
            call(s, lo, cnt)
        e1.record(stream)
        torch.cuda.synchronize()
        n_launch += iaat.iaat_launch_count() - n0
        res.setdefault(s.name(), [0.0, 0, s])
        res[s.name()][0] += e0.elapsed_time(e1) / args.steps
        res[s.name()][1] += cnt
    clk = clocks.stop()
    total_ms = sum(v[0] for v in res.values())
    total_ms = allreduce_max(total_ms, world)
    # strong scaling: the ranks share the fixed global batch; value = all
    # ranks' flops over the slowest rank's GEMM time
    flops = allreduce_sum(sum(v[2].flops(v[1]) for v in res.values()), world)
    value = flops / (total_ms * 1e-3) / 1e9
    pk = peaks()
    shapes_out = []
    for nm, (ms, cnt, s) in res.items():
        t = ms * 1e-3
        t_roof = max(s.flops(cnt) / (DMMA_PEAK_TFLOPS * 1e12), s.alg_bytes(cnt) / (pk["hbm_gbs"] * 1e9))
        shapes_out.append({"shape": nm, "batch": cnt, "ms": round(ms, 4), "gflops": round(s.flops(cnt) / t / 1e9, 1),
                           "frac_roofline": round(t_roof / t, 4)})
    nm, (ms, cnt, s) = max(res.items(), key=lambda kv: kv[1][0])
    dom_roof = roofline_of(s, cnt, ms * 1e-3, pk)
    dom_roof["kernel"] = nm
    dom_roof["share_of_step"] = round(ms / total_ms, 4)
    return {"metric": METRIC, "value": round(value, 1), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(total_ms, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "per_gpu": round(value / world, 1),
            "config": {"workload": desc, "global_batch": shapes[0].batch,
                       "parallelism": "dp%d: contiguous shards of the fixed global batch (dist.shard_range), "
                                      "no collective on the data path" % world},
            "roofline": dom_roof, "gpu_launches": int(n_launch), "clocks": clk,
            "shapes": shapes_out}


def run_e2e(args, chunks, bufs, call, stream, world):
    """Same sweep through the public C ABI, inputs from pinned host memory:
    H2D of A, B, C and D2H of C per call are inside the timed region.
    Copies are pipelined the way a user would: an upload stream, the compute
    stream and a download stream, so that the H2D of call i+1, the GEMM of
    call i and the D2H of call i-1 overlap (PCIe is full duplex)."""
    import torch
    host = {}
    for key, (A, B, C) in bufs.items():
        # pinned host copies filled straight from the device (no pageable
        # intermediate: one rank per GPU would otherwise double its host RAM)
        hs = []
        for t in (A, B, C):
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t)
            hs.append(h)
        host[key] = tuple(hs)
    steps = max(1, min(args.steps, args.e2e_steps))
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    last_down = [None]

    def step():
        h2d = d2h = 0
        for s, lo, cnt in chunks:
            key = (s.dtype, s.M, s.N, s.K, s.tr, cnt)
            (A, B, C), (hA, hB, hC) = bufs[key], host[key]
            with torch.cuda.stream(up):
                if last_down[0] is not None:
                    up.wait_event(last_down[0])  # previous step's reads of these buffers are done
                A.copy_(hA, non_blocking=True)
                B.copy_(hB, non_blocking=True)
                C.copy_(hC, non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(up)
            stream.wait_event(ev_in)
            call(s, lo, cnt)
            ev_out = torch.cuda.Event()
            ev_out.record(stream)
            with torch.cuda.stream(down):
                down.wait_event(ev_out)
                hC.copy_(C, non_blocking=True)
            h2d += (A.numel() + B.numel() + C.numel()) * A.element_size()
            d2h += C.numel() * C.element_size()
        ev = torch.cuda.Event()
        ev.record(down)
        last_down[0] = ev
        return h2d, d2h

    step()
    torch.cuda.synchronize()
    barrier(world)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    up.wait_stream(stream)
    for _ in range(steps):
        h2d, d2h = step()
    stream.wait_stream(down)
    stream.wait_stream(up)
    t1.record(stream)
    torch.cuda.synchronize()
    ms = allreduce_max(t0.elapsed_time(t1) / steps, world)
    flops = sum(s.flops(cnt) for s, lo, cnt in chunks)
    return {"value": round(flops * world / (ms * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": steps,
            "ms_per_step": round(ms, 3), "pipelined": "upload / compute / download streams"}


# ---------------------------------------------------------------- CPU oracle (baseline / reference arm)
def oracle_sample(shapes, frac):
    out = []
    for s in shapes:
        out.append((s, max(1, int(s.batch * frac))))
    return out


def run_oracle_timed(shapes, frac, repeats=1):
    import datagen
    import oracle
    dt = {"f32": np.float32, "f64": np.float64, "c32": np.float32, "c64": np.float64}
    cdt = {"c32": np.complex64, "c64": np.complex128}
    sample = oracle_sample(shapes, frac)
    inputs = []
    for s, n in sample:
        ra, ca, rb, cb = s.stored()
        ids = np.arange(n)
        w = 2 if s.cplx else 1
        A = datagen.fill_host(s.seed, 0, dt[s.dtype], w * ra, ca, w * ra, w * ra * ca, ids)
        B = datagen.fill_host(s.seed, 1, dt[s.dtype], w * rb, cb, w * rb, w * rb * cb, ids)
        C = datagen.fill_host(s.seed, 2, dt[s.dtype], w * s.M, s.N, w * s.M, w * s.M * s.N, ids)
        if s.cplx:
            A, B, C = A.view(cdt[s.dtype]), B.view(cdt[s.dtype]), C.view(cdt[s.dtype])
        inputs.append((s, n, A, B, C))
    total_t, total_f, threads = 0.0, 0.0, 0
    for _ in range(repeats):
        for s, n, A, B, C in inputs:
            ra, ca, rb, cb = s.stored()
            t = time.perf_counter()
            fn = oracle.ref_cgemm if s.cplx else oracle.ref_gemm
            _, _, threads = fn(s.tr[0], s.tr[1], s.M, s.N, s.K, s.alpha, A, ra, ra * ca, B, rb,
                               rb * cb, s.beta, C, s.M, s.M * s.N, n, want_den=False)
            total_t += time.perf_counter() - t
            total_f += s.flops(n)
    return total_f / total_t / 1e9, threads, total_t


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_oracle_one_thread(shapes, frac):
    """Per-core figure: the same oracle on ONE host thread, on a
    small prefix of every shape's batch."""
    import datagen
    import oracle
    dt = {"f32": np.float32, "f64": np.float64}
    tt, ff = 0.0, 0.0
    for s in shapes:
        if s.cplx:
            continue
        n = max(1, int(s.batch * frac))
        ra, ca, rb, cb = s.stored()
        ids = np.arange(n)
        A = datagen.fill_host(s.seed, 0, dt[s.dtype], ra, ca, ra, ra * ca, ids)
        B = datagen.fill_host(s.seed, 1, dt[s.dtype], rb, cb, rb, rb * cb, ids)
        C = datagen.fill_host(s.seed, 2, dt[s.dtype], s.M, s.N, s.M, s.M * s.N, ids)
        t = time.perf_counter()
        oracle.ref_gemm(s.tr[0], s.tr[1], s.M, s.N, s.K, s.alpha, A, ra, ra * ca, B, rb, rb * cb, s.beta, C,
                        s.M, s.M * s.N, n, nthreads=1, want_den=False)
        tt += time.perf_counter() - t
        ff += s.flops(n)
    return ff / tt / 1e9 if tt > 0 else None, frac


def run_cpu_baseline(shapes, args):
    frac = args.cpu_frac
    gf, threads, t = run_oracle_timed(shapes, frac)
    gf1, frac1 = run_oracle_one_thread(shapes, frac / 64)
    return {"value": round(gf, 3), "unit": "GFLOP/s", "cores": threads, "kind": "oracle",
            "cpu_model": cpu_model(), "one_thread_gflops": round(gf1, 3) if gf1 else None,
            "sample": "first %.4g of every shape's batch of the same step (all %d calls), fp64-accumulating "
                      "C triple loop, OpenMP over problems; %.1f s of CPU time; one_thread: first %.4g on 1 thread"
                      % (frac, len(shapes), t, frac1)}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return None
    shapes, desc = workload(args.config)
    frac = args.cpu_frac
    run_oracle_timed(shapes, frac / 4)  # warm-up (untimed)
    vals = []
    t_all = 0.0
    threads = 0
    for _ in range(max(1, args.steps)):
        gf, threads, t = run_oracle_timed(shapes, frac)
        vals.append(gf)
        t_all += t
    value = float(np.median(vals))
    sample = ("first %.4g of every shape's batch per step (%d calls), CPU oracle oracle/ref_gemm.c, "
              "OpenMP over problems" % (frac, len(shapes)))
    return {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_all / max(1, args.steps) * 1e3, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if shapes[0].dtype == "f32" else "f64", "data": "synthetic",
            "config": {"workload": desc, "parallelism": "host cores (OpenMP)"},
            "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": threads, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ---------------------------------------------------------------- distributed plumbing
_PG = None


def init_dist():
    global _PG
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
        _PG = dist
    return rank, world, local


def barrier(world):
    if world > 1 and _PG is not None:
        _PG.barrier()


def allreduce_max(x, world):
    if world > 1 and _PG is not None:
        import torch
        dev = "cuda" if torch.cuda.is_available() and _PG.get_backend() == "nccl" else "cpu"
        t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
        _PG.all_reduce(t, op=_PG.ReduceOp.MAX)
        return float(t.item())
    return float(x)


def allreduce_sum(x, world):
    if world > 1 and _PG is not None:
        import torch
        dev = "cuda" if torch.cuda.is_available() and _PG.get_backend() == "nccl" else "cpu"
        t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
        _PG.all_reduce(t, op=_PG.ReduceOp.SUM)
        return float(t.item())
    return float(x)


def load_traffic(name, batch):
    """dram bytes per launch of exactly this launch (shape AND batch) from a
    committed ncu --set full capture (profiles/traffic.json, key
    "<shape>@<batch>"), else None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("%s@%d" % (name, batch))
    except Exception:
        return None


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2,
                    help="BASELINE.json configs 1-5; 6/7 = complex fp32/fp64 sweeps (SURVEY f1); "
                         "8/9 = fp32 TN above 32^3, fp64 TN/TT (SURVEY f2); 10 = held-out n = 2 (mod 4) squares")
    ap.add_argument("--cpu-frac", type=float, default=0.5)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--grouped", action="store_true",
                    help="run the workload as one grouped (variable-size) call per step (SURVEY f4)")
    args = ap.parse_args(argv)
    env_world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus != env_world:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%d: launch N>1 with "
                         "torch.distributed.run --nproc-per-node N ... --gpus N" % (args.gpus, env_world))
    rank, world, local = init_dist()
    if args.impl == "reference":
        line = run_reference_arm(args, rank, world)
    else:
        line = run_ours(args, rank, world, local)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1 and _PG is not None:
        _PG.barrier()
        _PG.destroy_process_group()


if __name__ == "__main__":
    main()
