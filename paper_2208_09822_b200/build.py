"""Build libiaat.so in-tree: install-time generation + nvcc for sm_100a.

    python -m paper_2208_09822_b200.build [--force] [-j N]

1. gen/generate.py writes the kernel array (csrc/gen/*.cu, catalog.inc,
   kernel_table.inc) -- the paper's install-time stage.
2. nvcc compiles every translation unit for sm_100a only
   (-gencode arch=compute_100a,code=sm_100a -lineinfo, no fast-math), in
   parallel, and links paper_2208_09822_b200/libiaat.so (static cudart).
   ptxas register/spill reports are kept in build/ptxas_<unit>.log.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "iaat")
LIB = os.path.join(PKG, "libiaat.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                "-I" + CSRC, "-I" + os.path.join(ROOT, "include")]


def _headers():
    out = []
    for d in (CSRC, os.path.join(CSRC, "gen"), os.path.join(ROOT, "include")):
        if os.path.isdir(d):
            out += sorted(os.path.join(d, f) for f in os.listdir(d) if f.endswith((".h", ".cuh", ".inc")))
    return out


def _digest(src, headers):
    h = hashlib.sha256()
    for p in [src] + headers:
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(FLAGS).encode())
    return h.hexdigest()


def _compile(src, headers, force):
    name = os.path.basename(src)
    obj = os.path.join(BUILD, name + ".o")
    stamp = obj + ".sha"
    dig = _digest(src, headers)
    if not force and os.path.exists(obj) and os.path.exists(stamp) and open(stamp).read() == dig:
        return obj, False
    cmd = [NVCC] + FLAGS + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(os.path.join(BUILD, "ptxas_%s.log" % name), "w") as f:
        f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed for %s:\n%s" % (src, r.stderr[-4000:]))
    with open(stamp, "w") as f:
        f.write(dig)
    return obj, True


def build(force: bool = False, jobs: int = 0, verbose: bool = True) -> str:
    sys.path.insert(0, os.path.join(PKG, "gen"))
    import generate  # noqa: E402
    sys.path.pop(0)
    gen_files = generate.main([])
    os.makedirs(BUILD, exist_ok=True)
    headers = _headers()
    srcs = [os.path.join(CSRC, "api.cu"), os.path.join(CSRC, "planner.cpp")] + sorted(gen_files)
    jobs = jobs or max(1, os.cpu_count() or 1)
    changed = False
    objs = []
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        futs = [ex.submit(_compile, s, headers, force) for s in srcs]
        for f in futs:
            o, ch = f.result()
            objs.append(o)
            changed |= ch
    if changed or force or not os.path.exists(LIB):
        tmp = LIB + ".tmp%d" % os.getpid()
        subprocess.check_call([NVCC] + ARCH + ["-shared", "-o", tmp] + objs)
        os.replace(tmp, LIB)
        if verbose:
            print("built", LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=0)
    a = ap.parse_args()
    build(a.force, a.j)
