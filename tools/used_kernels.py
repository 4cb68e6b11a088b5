#!/usr/bin/env python3
"""Which generated kernels do the bench configs' plans (tuning table or cost
model) launch?  Cross-checked against the ptxas spill reports of the build:
    python tools/used_kernels.py [--configs 1 2 3 4 5 6 7]
Prints one line per used kernel with its spill bytes; exit 1 if any spills."""
import argparse
import glob
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def kernel_of(p, dt, tr):
    fam = p.get("family")
    if fam == "ksg":
        return "iaat_ksg_f32_%s_%dx%d_l%d_k%du%d_g%dw%d" % (tr, p["mr"], p["nr"], p["lane_rows"], p["kc"], p["ku"],
                                                           p["groups"], p["warps_per_group"])
    cls = p.get("classes") or []
    if fam == "ks1_fma":
        return "iaat_ks1_%s_%s_%dx%d" % (dt, tr, cls[0]["mr"], cls[0]["nr"])
    if fam == "ksu_fma":
        return "iaat_ksu_%s_%s_%dx%d" % (dt, tr, cls[0]["mr"], cls[0]["nr"])
    if fam == "ks_dmma":
        pre = "ksz" if dt == "c64" else "ksd"
        return "iaat_%s_%s_%s_%dx%d" % (pre, dt, tr, cls[0]["mr"] // 8, cls[0]["nr"] // 8)
    if fam == "ks_fma":
        return "iaat_ks_%s_%s" % (dt, tr)
    return "iaat_%s_%s_v%d" % (dt, tr, p.get("vec", 0))


def spills():
    out = {}
    for lg in glob.glob(os.path.join(ROOT, "build", "iaat", "ptxas_*.log")):
        txt = open(lg).read()
        for m in re.finditer(r"Compiling entry function '(\w+)'.*?(\d+) bytes spill stores, (\d+) bytes spill loads",
                             txt, re.S):
            name = re.sub(r"^_ZN4iaat\d+", "", m.group(1)).split("E14CUtensor")[0].split("E11Iaat")[0]
            out[name] = (int(m.group(2)), int(m.group(3)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="*", default=[1, 2, 3, 4, 5, 6, 7])
    a = ap.parse_args()
    from paper_2208_09822_b200 import iaat
    from paper_2208_09822_b200.tune import config_shapes
    sp = spills()
    used = {}
    for cfg in a.configs:
        for dt, tr, M, N, K, batch, alpha, beta in config_shapes(cfg):
            d = {"f32": 0, "f64": 1, "c32": 2, "c64": 3}[dt]
            ra, ca = (M, K) if tr[0] == "N" else (K, M)
            rb, cb = (K, N) if tr[1] == "N" else (N, K)
            if cfg == 5:
                batch = min(batch, 700000)
            p = iaat.iaat_plan_describe(d, tr[0], tr[1], M, N, K, ra, ra * ca, rb, rb * cb, M, M * N, batch,
                                        beta == 0)
            used.setdefault(kernel_of(p, dt, tr), []).append("c%d:%s%dx%dx%d" % (cfg, tr, M, N, K))
    bad = 0
    for k in sorted(used):
        s = sp.get(k)
        flag = ""
        if s and (s[0] or s[1]):
            flag = "  SPILLS %d/%d B" % s
            bad += 1
        print("%-44s %3d inputs%s" % (k, len(used[k]), flag))
    print("%d used kernels, %d spill" % (len(used), bad))
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
