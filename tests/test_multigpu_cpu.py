"""Multi-GPU path on CPU: world-size-2 gloo processes shard a batch by
contiguous ranges (paper_2208_09822_b200.dist), each computes its shard with
the CPU oracle standing in for its GPU, and the gathered result must equal the
unsharded computation bitwise; the bench's max-over-ranks timing reduction is
exercised over the same process group.  No collective touches the data path
in the product -- the all_gather here is only the test's check."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2208_09822_b200.dist import aggregate_gflops, shard_range, weak_range


def test_shard_range_partitions():
    for total in (0, 1, 7, 2_000_000, 12345):
        for world in (1, 2, 3, 4, 8):
            cuts = [shard_range(total, r, world) for r in range(world)]
            assert cuts[0][0] == 0 and cuts[-1][1] == total
            for (a, b), (c, d) in zip(cuts[:-1], cuts[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in cuts]
            assert max(sizes) - min(sizes) <= 1
    assert weak_range(100, 3) == (300, 400)
    assert aggregate_gflops([2e9, 2e9], [1.0, 2.0]) == 2.0
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import datagen
    import oracle
    M, N, K, total = 7, 5, 9, 101
    lo, hi = shard_range(total, rank, world)
    ids = np.arange(lo, hi)
    A = datagen.fill_host(3, 0, np.float32, M, K, M, M * K, ids)
    B = datagen.fill_host(3, 1, np.float32, K, N, K, K * N, ids)
    C = datagen.fill_host(3, 2, np.float32, M, N, M, M * N, ids)
    ref, _, _ = oracle.ref_gemm("N", "N", M, N, K, 1.5, A, M, M * K, B, K, K * N, 0.5, C, M, M * N, len(ids),
                                nthreads=1)
    # pad to equal length for all_gather
    maxn = max(shard_range(total, r, world)[1] - shard_range(total, r, world)[0] for r in range(world))
    buf = torch.full((maxn, N, M), float("nan"), dtype=torch.float64)
    buf[:len(ids)] = torch.from_numpy(ref)
    gathered = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(gathered, buf)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # bench.py's max-over-ranks time
    if rank == 0:
        parts = []
        for r in range(world):
            a, b = shard_range(total, r, world)
            parts.append(gathered[r][:b - a].numpy())
        out.put((np.concatenate(parts), float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_shards_match_unsharded():
    import datagen
    import oracle
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    sharded, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    M, N, K, total = 7, 5, 9, 101
    ids = np.arange(total)
    A = datagen.fill_host(3, 0, np.float32, M, K, M, M * K, ids)
    B = datagen.fill_host(3, 1, np.float32, K, N, K, K * N, ids)
    C = datagen.fill_host(3, 2, np.float32, M, N, M, M * N, ids)
    ref, _, _ = oracle.ref_gemm("N", "N", M, N, K, 1.5, A, M, M * K, B, K, K * N, 0.5, C, M, M * N, total)
    assert np.array_equal(sharded, ref)
    assert tmax == 2.0


def test_bench_reference_arm_under_torchrun_world2():
    """bench.py launched the way the driver launches N > 1 (torchrun, one
    process per rank, 127.0.0.1 rendezvous), here on CPU with gloo: rank 0
    alone runs the reference arm and prints exactly one JSON line; rank 1
    exits 0 without work."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--config", "1",
           "--cpu-frac", "0.01"]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=root, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


def _config5_worker(rank, world, port, out):
    """The bench's own config-5 sharding code path (bench.plan_chunks) on one
    gloo rank: the chunks it would call, their generated inputs (global ids)
    and the oracle's results on a sample of them, gathered to rank 0."""
    import sys
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    import datagen
    import oracle
    shapes, _ = bench.workload(5)
    # a small stand-in HBM so that every shape is also chunked inside a shard
    chunks = bench.plan_chunks(shapes, 5, rank, world, hbm_cap=64 << 20)
    spans = [(s.name(), lo, cnt) for s, lo, cnt in chunks]
    # inputs + results of the first and last problem of every chunk (the
    # shard / chunk boundaries), fp64 n = 16 shapes only (oracle cost)
    res = []
    for s, lo, cnt in chunks:
        if s.M != 16:
            continue
        for g in (lo, lo + cnt - 1):
            ids = np.array([g])
            A = datagen.fill_host(s.seed, 0, np.float64, 16, 16, 16, 256, ids)
            B = datagen.fill_host(s.seed, 1, np.float64, 16, 16, 16, 256, ids)
            ref, _, _ = oracle.ref_gemm(s.tr[0], s.tr[1], 16, 16, 16, 1.0, A, 16, 256, B, 16, 256, 0.0, None, 16,
                                        256, 1, nthreads=1)
            res.append((s.name(), g, ref))
    allspans = [None] * world
    allres = [None] * world
    dist.all_gather_object(allspans, spans)
    dist.all_gather_object(allres, res)
    if rank == 0:
        out.put((allspans, allres))
    dist.barrier()
    dist.destroy_process_group()


def test_config5_strong_scaling_shards_under_gloo_world2():
    """Row e (BASELINE config 5): under world size 2 the bench
    shards the FIXED global batch of 2,000,000 into contiguous per-rank
    ranges (dist.shard_range), chunked, disjoint and covering every problem
    exactly once; the shard-boundary problems' inputs (generated by global
    id) and oracle results equal the unsharded ones bitwise."""
    import datagen
    import oracle
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_config5_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    allspans, allres = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    per_shape = {}
    for r, spans in enumerate(allspans):
        lo_r, hi_r = shard_range(2_000_000, r, world)
        for name, lo, cnt in spans:
            assert lo_r <= lo and lo + cnt <= hi_r, (r, name, lo, cnt)
            per_shape.setdefault(name, []).append((lo, cnt))
    assert len(per_shape) == 12
    for name, sp in per_shape.items():
        sp.sort()
        assert sp[0][0] == 0 and sum(c for _, c in sp) == 2_000_000
        for (a, c), (b, _) in zip(sp[:-1], sp[1:]):
            assert a + c == b, name
    n = 0
    for res in allres:
        for name, g, ref in res:
            tr = name.split("_")[1]
            ids = np.array([g])
            A = datagen.fill_host(4, 0, np.float64, 16, 16, 16, 256, ids)
            B = datagen.fill_host(4, 1, np.float64, 16, 16, 16, 256, ids)
            one, _, _ = oracle.ref_gemm(tr[0], tr[1], 16, 16, 16, 1.0, A, 16, 256, B, 16, 256, 0.0, None, 16, 256, 1,
                                        nthreads=1)
            assert np.array_equal(one, ref), (name, g)
            n += 1
    assert n >= 8


def test_bench_rejects_gpus_world_mismatch():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=120, cwd=root,
                       env=dict(os.environ, WORLD_SIZE="1"))
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stderr + r.stdout)
