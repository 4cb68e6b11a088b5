#!/usr/bin/env python3
"""Per-case register / spill report of the K-streamed kernels: compiles one
translation unit per (dtype, trans, mr, nr) catalog entry (a one-case
dispatch) with ptxas -v.  Used to bound the KS catalog (generate.py).

    python tools/ks_regs.py f32 NN [TT ...]
"""
import concurrent.futures as cf
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2208_09822_b200", "gen"))
import generate as g  # noqa: E402

CSRC = os.path.join(ROOT, "paper_2208_09822_b200", "csrc")


def one(dt, tr, mr, nr, unr, out):
    T = g.DTYPES[dt]
    ta = "true" if tr[0] == "T" else "false"
    tb = "true" if tr[1] == "T" else "false"
    src = """#include "iaat_ks.cuh"
namespace iaat {
struct D {
    static __device__ __forceinline__ void run(const IaatKsParams &p, const IaatClass &c, unsigned char *smem,
                                               uint64_t *full, uint64_t *empty, int warp, int lane)
    {
        ks_fma_class_loop<%s, %s, %s, %d, %d, %d>(p, c, smem, full, empty, warp, lane);
    }
};
__global__ void __launch_bounds__(%s, 1)
kcase(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
      const __grid_constant__ IaatKsParams p)
{
    ks_kernel_body<%s, %s, %s, D, true>(&tmA, &tmB, p);
}
}
""" % (T, ta, tb, mr, nr, unr, "IAAT_MAX_THREADS", T, ta, tb)
    fn = os.path.join(out, "c_%s_%s_%d_%d_%d.cu" % (dt, tr, mr, nr, unr))
    open(fn, "w").write(src)
    r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xptxas", "-v",
                        "-I" + CSRC, "-I" + os.path.join(ROOT, "include"), "-c", fn, "-o", fn + ".o"],
                       capture_output=True, text=True)
    txt = r.stdout + r.stderr
    regs = re.search(r"Used (\d+) registers", txt)
    sps = re.findall(r"(\d+) bytes spill stores, (\d+) bytes spill loads", txt)
    sp = max(sps, key=lambda x: int(x[0])) if sps else None
    return (dt, tr, mr, nr, unr, int(regs.group(1)) if regs else -1, int(sp[0]) if sp else -1)


def main():
    args = sys.argv[1:]
    jobs = []
    for i in range(0, len(args), 2):
        dt, tr = args[i], args[i + 1]
        unrs = [int(x) for x in os.environ.get("KS_UNR", "0").split(",")]
        for mr, nr in sorted(set(g.ks_fma_tiles(dt, tr) + g.KS1_TILES[dt])):
            if mr * nr >= 1:
                for u in unrs:
                    jobs.append((dt, tr, mr, nr, u or g.ks_unroll(dt, tr, mr, nr)))
    out = os.environ.get("KS_UNR_OUT")
    table = {}
    if out and os.path.exists(out):
        table = json.load(open(out))
    res = []
    with cf.ThreadPoolExecutor(os.cpu_count()) as ex:
        for r in ex.map(lambda j: one(*j, "/tmp/kscase"), jobs):
            print("%s %s %dx%d unr=%d regs=%d spill=%d" % r, flush=True)
            res.append(r)
    if out:
        # install-time register check: the deepest spill-free k-block
        # buffering per catalog entry (generate.py reads this table)
        best = {}
        for dt, tr, mr, nr, unr, regs, spill in res:
            k = "%s_%s_%dx%d" % (dt, tr, mr, nr)
            # spill-free double buffering if possible; a single-buffered entry
            # may keep a few spilled words outside the k loop (<= 64 B)
            if spill == 0 or (unr == 1 and spill <= 64):
                best[k] = max(best.get(k, 0), unr)
            else:
                best.setdefault(k, 0)  # 0: spills at every buffering depth -> not in the catalog
        table.update(best)
        with open(out, "w") as f:
            json.dump(table, f, indent=0, sort_keys=True)


if __name__ == "__main__":
    main()
