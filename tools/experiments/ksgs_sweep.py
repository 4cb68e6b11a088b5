"""Time every ksgs entry (forced) at several ring depths on given shapes.

    python tools/experiments/ksgs_sweep.py NN 37x67x79 61x67x31 ...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2208_09822_b200 import iaat, tune  # noqa: E402

tr = sys.argv[1]
beta = float(os.environ.get("BETA", "1.0"))
for arg in sys.argv[2:]:
    M, N, K = (int(x) for x in arg.split("x"))
    b = tune.Bench("f32", tr, M, N, K, 100000, 1.0, beta)
    tune.set_knobs()
    base = b.time_us()
    p0 = b.plan()
    print("%s %s batch=%d default %.1f us  plan=%s" % (tr, arg, b.batch, base,
          {k: p0.get(k) for k in ("family", "entry", "mr", "nr", "P", "S")}), flush=True)
    for e in iaat.iaat_catalog_describe():
        if e["family"] != "ksgs" or e["trans"] != tr:
            continue
        tune.set_knobs(family=8, order=e["index"])
        p = b.plan()
        if p.get("family") != "ksgs" or p.get("entry") != e["index"]:
            continue
        smax = p["S"]
        for s in sorted({smax, max(1, smax - 1), max(1, smax - 2), e["g"] + 2, e["g"] + 1}):
            if s > smax:
                continue
            tune.set_knobs(family=8, order=e["index"], s=s)
            us = b.time_us()
            print("  e%-2d %dx%d l%d g%dw%d Mv=%d Nv=%d P=%d S=%d: %.1f us (%.2fx)" % (
                e["index"], e["mr"], e["nr"], e["lr"], e["g"], e["w"], p["Mv"], p["Nv"], p["P"], s, us,
                base / us), flush=True)
    tune.set_knobs()
    b.free()
