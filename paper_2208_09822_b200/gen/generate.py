#!/usr/bin/env python3
"""Install-time stage: generate the kernel array (Sec. III-A/IV).

The paper's install-time stage auto-generates "hundreds of kernels of
different sizes" (Table I) -- one fixed-size kernel per block
size C_c = m_c x n_c, type and transposition -- which the run-time stage then
invokes directly ("kernel array").  On B200 the analogue is:

* the catalog: every exact micro-tile size (mr, nr) a thread (FMA family) or
  a warp (DMMA family, fp64) computes, per dtype and transposition.  Table I's
  sizes came from 32 x 128-bit NEON registers and do not
  transfer; the GPU catalog is bounded by the accumulator-register budget
  (mr*nr*(elt/4) <= 64 registers, no spills -- checked by tests/test_build.py
  through `nvcc -Xptxas -v`);
* one persistent pipeline kernel per (dtype, transA, transB, vec) whose
  warp-uniform dispatch switch lists the catalog entries (the generated
  "kernel array"), instantiated from the templates in csrc/iaat_device.cuh;
* a launch table the run-time planner indexes.

Writes csrc/gen/{catalog.inc, kernel_table.inc, k_<dt>_<tr>_v<vec>.cu}.
"""
from __future__ import annotations

import argparse
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(os.path.dirname(HERE), "csrc")
OUT = os.path.join(CSRC, "gen")

DTYPES = {"f32": "float", "f64": "double"}
TRANS = ["NN", "NT", "TN", "TT"]
MAX_MR = 8
MAX_NR = 8
# fp64 DMMA warp tiles: (wm, wn) DMMA.8x8x4 blocks per warp
DMMA_TILES = [(1, 1), (1, 2), (2, 1), (2, 2), (2, 4), (4, 2), (4, 4)]


def dmma_tiles(tr):
    """DMMA warp tiles (wm x wn blocks of 8x8) for a transposition; 4x4 would
    spill in TN (both fragments loaded as 16-byte pairs plus 64 accumulators)."""
    return [t for t in DMMA_TILES if not (tr == "TN" and t == (4, 4))]


def fma_code(mr, nr):
    return (mr - 1) * MAX_NR + (nr - 1)


def dmma_code(wm, wn):
    return 100 + 10 * wm + wn


KU = {"f32": 4, "f64": 2}  # k-steps per unrolled block = one 16 B vector (csrc/iaat_device.cuh)
# 32-bit registers for accumulators + live operand fragments (fp64 lower:
# 64-bit address/pointer temporaries of the DFMA tiles also compete)
REG_BUDGET = {"f32": 112, "f64": 100}


def fma_regs(dt, tr, mr, nr):
    """Registers the C_c block and the operand fragments of one k-block need
    -- the register allocator's budget (A_c / B_c / C_c
    register groups), with nvcc doing the allocation.  An operand contiguous
    along k is loaded KU k-steps at a time, so KU fragments are live."""
    words = 1 if dt == "f32" else 2
    a_kcontig = tr[0] == "T"
    b_kcontig = tr[1] == "N"
    fa = KU[dt] * mr if a_kcontig else mr
    fb = KU[dt] * nr if b_kcontig else nr
    return words * (mr * nr + fa + fb)


def fma_unroll(dt, tr, mr, nr):
    """k-block unroll (ping-pang): 2 when two blocks of fragments plus the
    accumulators still fit the register budget, else 1."""
    words = 1 if dt == "f32" else 2
    base = fma_regs(dt, tr, mr, nr)
    frags = base // words - mr * nr
    return 2 if words * (mr * nr + 2 * frags) <= REG_BUDGET[dt] else 1


def fma_tiles(dt, tr=None):
    """Catalog of exact FMA micro-tiles for (dtype, trans): all (mr, nr) up to
    8 x 8 whose registers fit the budget (no spills; checked by
    tests/test_build.py with `nvcc -Xptxas -v`).  tr=None: union."""
    trs = [tr] if tr else TRANS
    return [(mr, nr) for mr in range(1, MAX_MR + 1) for nr in range(1, MAX_NR + 1)
            if any(fma_regs(dt, t, mr, nr) <= REG_BUDGET[dt] - TRANS_MARGIN[dt].get(t, 0) for t in trs)]


# measured (ptxas -v): TT's paired FFMA2 accumulators with both fragments
# 16 bytes along k leave less room -- its 8 x 8 entry spilled
TRANS_MARGIN = {"f32": {"TT": 12}, "f64": {}}


def catalog():
    ents = []
    for dt in DTYPES:
        for tr in TRANS:
            for mr, nr in fma_tiles(dt, tr):
                ents.append({"family": "fma", "dtype": dt, "trans": tr, "mr": mr, "nr": nr,
                             "code": fma_code(mr, nr)})
        for tr in TRANS:
            for mr, nr in ks_fma_tiles(dt, tr):
                ents.append({"family": "ks_fma", "dtype": dt, "trans": tr, "mr": mr, "nr": nr,
                             "code": fma_code(mr, nr)})
            for mr, nr in ks1_tiles(dt, tr):
                ents.append({"family": "ks1_fma", "dtype": dt, "trans": tr, "mr": mr, "nr": nr,
                             "code": fma_code(mr, nr)})
        if dt == "f64":
            for tr in TRANS:
                for wm, wn in KSD_TILES:
                    ents.append({"family": "ks_dmma", "dtype": dt, "trans": tr, "mr": 8 * wm, "nr": 8 * wn,
                                 "code": dmma_code(wm, wn)})
            for tr in TRANS:
                for wm, wn in dmma_tiles(tr):
                    ents.append({"family": "dmma", "dtype": dt, "trans": tr, "mr": 8 * wm,
                                 "nr": 8 * wn, "code": dmma_code(wm, wn)})
    return ents


def kernel_name(dt, tr, vec):
    return "iaat_%s_%s_v%d" % (dt, tr, vec)


def gen_kernel_file(dt, tr, vec):
    T = DTYPES[dt]
    ta = "true" if tr[0] == "T" else "false"
    tb = "true" if tr[1] == "T" else "false"
    v = "true" if vec else "false"
    name = kernel_name(dt, tr, vec)
    cases = []
    for mr, nr in fma_tiles(dt, tr):
        cases.append("        case %d: fma_class_loop<%s, %s, %s, %d, %d, %s, %d>(p, c, smem, full, empty, warp, lane); break;"
                     % (fma_code(mr, nr), T, ta, tb, mr, nr, v, fma_unroll(dt, tr, mr, nr)))
    if dt == "f64":
        for wm, wn in dmma_tiles(tr):
            cases.append("        case %d: dmma_class_loop<%s, %s, %d, %d, %s>(p, c, smem, full, empty, warp, lane); break;"
                         % (dmma_code(wm, wn), ta, tb, wm, wn, v))
    inc = '#include "../iaat_device.cuh"\n'
    if dt == "f64":
        inc += '#include "../iaat_dmma.cuh"\n'
    return """// GENERATED by gen/generate.py -- do not edit.  Kernel array entry for
// dtype=%(dt)s trans=%(tr)s vec=%(vec)d (install-time stage, PAPER.md:74-105).
%(inc)s
namespace iaat {
namespace {
struct Dispatch_%(name)s {
    static __device__ __forceinline__ void run(const IaatKParams &p, const IaatClass &c,
                                               unsigned char *smem, uint64_t *full,
                                               uint64_t *empty, int warp, int lane)
    {
        switch (c.code) {
%(cases)s
        default: __trap();
        }
    }
};
}  // namespace

__global__ void __launch_bounds__(IAAT_MAX_THREADS, 1) %(name)s(const __grid_constant__ IaatKParams p)
{
    pipeline_kernel_body<%(T)s, Dispatch_%(name)s>(p);
}

cudaError_t launch_%(name)s(const IaatKParams &p, int grid, int block, int smem, cudaStream_t s)
{
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(%(name)s, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             IAAT_SMEM_LIMIT);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    %(name)s<<<grid, block, smem, s>>>(p);
    return cudaGetLastError();
}
}  // namespace iaat
""" % {"dt": dt, "tr": tr, "vec": vec, "inc": inc, "name": name, "cases": "\n".join(cases), "T": T}


def ks_fma_tiles(dt, tr):
    """K-streamed multi-class kernel (one warp-uniform switch over the tile
    classes of a plan): the tiles whose inlined cases keep the whole kernel
    spill-free under the 128-register bound (tests/test_build.py)."""
    lim = KS_MULTI_MAX_AREA[dt] // (2 if tr == "TN" else 1)  # TN: both operands K-major
    return [(mr, nr) for mr in range(1, MAX_MR + 1) for nr in range(1, MAX_NR + 1)
            if mr * nr <= lim and ks_unroll(dt, tr, mr, nr) > 0]


def ks1_tiles(dt, tr):
    return [t for t in KS1_TILES[dt] if ks_unroll(dt, tr, *t) > 0]


KS_MULTI_MAX_AREA = {"f32": 24, "f64": 8}
# single-class kernels (one exact tile class covers the whole C): each is its
# own kernel, so each gets its own register allocation -- the big tiles live
# here (tools/ks_regs.py checks them one by one)
KS1_TILES = {
    "f32": [(2, 4), (4, 2), (2, 8), (8, 2), (3, 8), (8, 3), (4, 4), (4, 5), (5, 4), (4, 6), (6, 4), (4, 7), (7, 4),
            (4, 8), (8, 4), (5, 5), (5, 8), (8, 5), (6, 6), (6, 8), (8, 6), (7, 8), (8, 7), (8, 8)],
    "f64": [(2, 2), (2, 4), (4, 2), (2, 8), (8, 2), (4, 4), (4, 8), (8, 4)],
}


_KS_UNROLL = None


# fp64 DMMA warp tiles of the K-streamed family: (wm, wn) blocks of 8 x 8,
# accumulators 4*wm*wn registers <= 64
KSD_TILES = [(wm, wn) for wm in range(1, 6) for wn in range(1, 6) if wm * wn <= 16]


def ksd_kernel_name(tr, wm, wn):
    return "iaat_ksd_f64_%s_%dx%d" % (tr, wm, wn)


def gen_ksd_file(tr):
    """Single-class K-streamed DMMA kernels (fp64) of one transposition."""
    ta = "true" if tr[0] == "T" else "false"
    tb = "true" if tr[1] == "T" else "false"
    parts = []
    for wm, wn in KSD_TILES:
        name = ksd_kernel_name(tr, wm, wn)
        parts.append("""
struct Dispatch_%(name)s {
    static __device__ __forceinline__ void run(const IaatKsParams &p, const IaatClass &c,
                                               unsigned char *smem, uint64_t *full,
                                               uint64_t *empty, int warp, int lane)
    {
        ks_dmma_class_loop<%(ta)s, %(tb)s, %(wm)d, %(wn)d>(p, c, smem, full, empty, warp, lane);
    }
};

__global__ void __launch_bounds__(IAAT_MAX_THREADS, 1)
%(name)s(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
         const __grid_constant__ IaatKsParams p)
{
    ks_kernel_body<double, %(ta)s, %(tb)s, Dispatch_%(name)s, true>(&tmA, &tmB, p);
}
%(launch)s""" % {"name": name, "ta": ta, "tb": tb, "wm": wm, "wn": wn, "launch": KS_LAUNCH % {"name": name}})
    return """// GENERATED by gen/generate.py -- do not edit.  K-streamed DMMA (fp64 tensor-core)
// kernels, trans=%s (install-time stage, PAPER.md:74-105).
#include "../iaat_ks.cuh"

namespace iaat {
%s
}  // namespace iaat
""" % (tr, "".join(parts))


def ks_unroll(dt, tr, mr, nr):
    """k-block register buffering of a K-streamed entry: 2 = double-buffered
    (ping-pang), 1 = single, 0 = spills even single-buffered
    (entry left out).  Measured at install time by tools/ks_regs.py (ptxas
    -v on one-entry kernels) into gen/ks_unroll.json -- the analogue of the
    paper's register-allocator budget."""
    global _KS_UNROLL
    if _KS_UNROLL is None:
        p = os.path.join(HERE, "ks_unroll.json")
        _KS_UNROLL = json.load(open(p)) if os.path.exists(p) else {}
    return _KS_UNROLL.get("%s_%s_%dx%d" % (dt, tr, mr, nr), 1)


def ks_kernel_name(dt, tr):
    return "iaat_ks_%s_%s" % (dt, tr)


def ks1_kernel_name(dt, tr, mr, nr):
    return "iaat_ks1_%s_%s_%dx%d" % (dt, tr, mr, nr)


KS_LAUNCH = """
cudaError_t launch_%(name)s(const CUtensorMap &tmA, const CUtensorMap &tmB, const IaatKsParams &p,
                             int grid, int block, int smem, cudaStream_t s)
{
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(%(name)s, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             IAAT_SMEM_LIMIT);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    %(name)s<<<grid, block, smem, s>>>(tmA, tmB, p);
    return cudaGetLastError();
}
"""


def gen_ks_kernel_file(dt, tr):
    """K-streamed TMA family (csrc/iaat_ks.cuh): the multi-class kernel of
    one (dtype, transposition)."""
    T = DTYPES[dt]
    ta = "true" if tr[0] == "T" else "false"
    tb = "true" if tr[1] == "T" else "false"
    name = ks_kernel_name(dt, tr)
    cases = []
    for mr, nr in ks_fma_tiles(dt, tr):
        # single-buffered here: the union of the inlined cases is what ptxas allocates
        cases.append("        case %d: ks_fma_class_loop<%s, %s, %s, %d, %d, 1>(p, c, smem, full, empty, warp, lane); break;"
                     % (fma_code(mr, nr), T, ta, tb, mr, nr))
    return """// GENERATED by gen/generate.py -- do not edit.  K-streamed kernel array entry for
// dtype=%(dt)s trans=%(tr)s (install-time stage, PAPER.md:74-105).
#include "../iaat_ks.cuh"

namespace iaat {
namespace {
struct Dispatch_%(name)s {
    static __device__ __forceinline__ void run(const IaatKsParams &p, const IaatClass &c,
                                               unsigned char *smem, uint64_t *full,
                                               uint64_t *empty, int warp, int lane)
    {
        switch (c.code) {
%(cases)s
        default: __trap();
        }
    }
};
}  // namespace

__global__ void __launch_bounds__(IAAT_MAX_THREADS, 1)
%(name)s(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
         const __grid_constant__ IaatKsParams p)
{
    ks_kernel_body<%(T)s, %(ta)s, %(tb)s, Dispatch_%(name)s>(&tmA, &tmB, p);
}
%(launch)s
}  // namespace iaat
""" % {"dt": dt, "tr": tr, "name": name, "cases": "\n".join(cases), "T": T, "ta": ta, "tb": tb,
       "launch": KS_LAUNCH % {"name": name}}


def gen_ks1_file(dt, tr):
    """Single-class K-streamed kernels of one (dtype, transposition)."""
    T = DTYPES[dt]
    ta = "true" if tr[0] == "T" else "false"
    tb = "true" if tr[1] == "T" else "false"
    parts = []
    for mr, nr in ks1_tiles(dt, tr):
        name = ks1_kernel_name(dt, tr, mr, nr)
        parts.append("""
struct Dispatch_%(name)s {
    static __device__ __forceinline__ void run(const IaatKsParams &p, const IaatClass &c,
                                               unsigned char *smem, uint64_t *full,
                                               uint64_t *empty, int warp, int lane)
    {
        ks_fma_class_loop<%(T)s, %(ta)s, %(tb)s, %(mr)d, %(nr)d, %(unr)d>(p, c, smem, full, empty, warp, lane);
    }
};

__global__ void __launch_bounds__(%(lb)s, 1)
%(name)s(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
         const __grid_constant__ IaatKsParams p)
{
    ks_kernel_body<%(T)s, %(ta)s, %(tb)s, Dispatch_%(name)s, true>(&tmA, &tmB, p);
}
%(launch)s""" % {"name": name, "T": T, "ta": ta, "tb": tb, "mr": mr, "nr": nr, "launch": KS_LAUNCH % {"name": name},
                     "unr": ks_unroll(dt, tr, mr, nr), "lb": "IAAT_MAX_THREADS"})
    return """// GENERATED by gen/generate.py -- do not edit.  Single-class K-streamed kernels,
// dtype=%s trans=%s (install-time stage, PAPER.md:74-105).
#include "../iaat_ks.cuh"

namespace iaat {
%s
}  // namespace iaat
""" % (dt, tr, "".join(parts))


def gen_table():
    decl, rows = [], []
    for di, dt in enumerate(DTYPES):
        for tr in TRANS:
            for vec in (0, 1):
                n = kernel_name(dt, tr, vec)
                decl.append("cudaError_t launch_%s(const IaatKParams &, int, int, int, cudaStream_t);" % n)
    body = []
    for dt in DTYPES:
        tb = []
        for tr in TRANS:
            tb.append("{&launch_%s, &launch_%s}" % (kernel_name(dt, tr, 0), kernel_name(dt, tr, 1)))
        body.append("    {" + ", ".join(tb) + "}")
    ks_decl, ks_body, ks1, ksd = [], [], [], []
    for dt in DTYPES:
        for tr in TRANS:
            ks_decl.append("cudaError_t launch_%s(const CUtensorMap &, const CUtensorMap &, const IaatKsParams &, "
                           "int, int, int, cudaStream_t);" % ks_kernel_name(dt, tr))
            for mr, nr in ks1_tiles(dt, tr):
                ks_decl.append("cudaError_t launch_%s(const CUtensorMap &, const CUtensorMap &, const IaatKsParams &, "
                               "int, int, int, cudaStream_t);" % ks1_kernel_name(dt, tr, mr, nr))
                ks1.append("    {%d, %d, %d, %d, &launch_%s}," % (list(DTYPES).index(dt), TRANS.index(tr), mr, nr,
                                                                  ks1_kernel_name(dt, tr, mr, nr)))
            if dt == "f64":
                for wm, wn in KSD_TILES:
                    ks_decl.append("cudaError_t launch_%s(const CUtensorMap &, const CUtensorMap &, "
                                   "const IaatKsParams &, int, int, int, cudaStream_t);" % ksd_kernel_name(tr, wm, wn))
                    ksd.append("    {%d, %d, %d, &launch_%s}," % (TRANS.index(tr), wm, wn, ksd_kernel_name(tr, wm, wn)))
        ks_body.append("    {" + ", ".join("&launch_%s" % ks_kernel_name(dt, tr) for tr in TRANS) + "}")
    return ("// GENERATED by gen/generate.py -- launch table [dtype][trans NN,NT,TN,TT][vec]\n"
            "namespace iaat {\n" + "\n".join(decl) +
            "\ntypedef cudaError_t (*LaunchFn)(const IaatKParams &, int, int, int, cudaStream_t);\n"
            "static const LaunchFn kLaunch[2][4][2] = {\n" + ",\n".join(body) + "\n};\n" +
            "\n".join(ks_decl) +
            "\ntypedef cudaError_t (*KsLaunchFn)(const CUtensorMap &, const CUtensorMap &, const IaatKsParams &, "
            "int, int, int, cudaStream_t);\n"
            "static const KsLaunchFn kLaunchKs[2][4] = {\n" + ",\n".join(ks_body) + "\n};\n"
            "struct Ks1Entry { int dtype, trans, mr, nr; KsLaunchFn fn; };\n"
            "static const Ks1Entry kLaunchKs1[] = {\n" + "\n".join(ks1) + "\n};\n"
            "struct KsdEntry { int trans, wm, wn; KsLaunchFn fn; };\n"
            "static const KsdEntry kLaunchKsd[] = {\n" + "\n".join(ksd) + "\n};\n"
            "}  // namespace iaat\n")


def gen_catalog_inc(ents):
    lines = ["// GENERATED by gen/generate.py -- the install-time kernel catalog.",
             "#define IAAT_FMA_MAX_MR %d" % MAX_MR, "#define IAAT_FMA_MAX_NR %d" % MAX_NR,
             "#define IAAT_FMA_CODE(mr, nr) (((mr) - 1) * IAAT_FMA_MAX_NR + ((nr) - 1))",
             "#define IAAT_DMMA_CODE(wm, wn) (100 + 10 * (wm) + (wn))",
             "struct IaatCatalogEntry { int family; int dtype; int trans; int mr; int nr; int code; };",
             "static const IaatCatalogEntry kCatalog[] = {"]
    for e in ents:
        lines.append("    {%d, %d, %d, %d, %d, %d}," % ({"fma": 0, "dmma": 1, "ks_fma": 2, "ks_dmma": 3, "ks1_fma": 4}[e["family"]],
                                                        0 if e["dtype"] == "f32" else 1,
                                                        TRANS.index(e["trans"]),
                                                        e["mr"], e["nr"], e["code"]))
    lines.append("};")
    lines.append("static const char kCatalogJson[] = %s;" % json.dumps(json.dumps(ents)))
    return "\n".join(lines) + "\n"


def write_if_changed(path, text):
    if os.path.exists(path):
        with open(path) as f:
            if f.read() == text:
                return False
    with open(path, "w") as f:
        f.write(text)
    return True


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=OUT)
    args = ap.parse_args(argv)
    os.makedirs(args.out, exist_ok=True)
    ents = catalog()
    files = []
    write_if_changed(os.path.join(args.out, "catalog.inc"), gen_catalog_inc(ents))
    write_if_changed(os.path.join(args.out, "kernel_table.inc"), gen_table())
    for dt in DTYPES:
        for tr in TRANS:
            for vec in (0, 1):
                p = os.path.join(args.out, "k_%s_%s_v%d.cu" % (dt, tr, vec))
                write_if_changed(p, gen_kernel_file(dt, tr, vec))
                files.append(p)
            p = os.path.join(args.out, "ks_%s_%s.cu" % (dt, tr))
            write_if_changed(p, gen_ks_kernel_file(dt, tr))
            files.append(p)
            p = os.path.join(args.out, "ks1_%s_%s.cu" % (dt, tr))
            write_if_changed(p, gen_ks1_file(dt, tr))
            files.append(p)
            if dt == "f64":
                p = os.path.join(args.out, "ksd_f64_%s.cu" % tr)
                write_if_changed(p, gen_ksd_file(tr))
                files.append(p)
    return files


if __name__ == "__main__":
    for f in main():
        print(f)
