#!/usr/bin/env python3
"""Top stall sites of one ncu capture: python tools/ncu_src.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ic = [h.index(c) for c in cols]
data = []
tot = {c: 0 for c in cols}
for r in rows[2:]:
    try:
        s = int(r[iS])
    except ValueError:
        continue
    st = {c: int(r[i] or 0) for c, i in zip(cols, ic)}
    for c in cols:
        tot[c] += st[c]
    data.append((s, r[iE], r[0][-5:], r[1].strip()[:48], st))
T = sum(d[0] for d in data)
print("total samples", T, {k: round(v / T, 3) for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v})
for s, e, a, src, st in sorted(data, key=lambda d: -d[0])[:n]:
    top = sorted(((v, k[6:]) for k, v in st.items() if v), reverse=True)[:3]
    print("%5d %9s %s %-48s %s" % (s, e, a, src, top))
