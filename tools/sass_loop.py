#!/usr/bin/env python3
"""sass_loop.py -- instruction mix of the hottest loop of each kernel.

For every function in a cubin / object / executable (cuobjdump -sass), find
the innermost backward-branch body [target, branch] holding at least half
of the FFMA2/DMMA of the busiest loop
and print that body's instruction counts (FFMA2, LDS, MOV, other) and the
instructions per FFMA2.  Used to spot register shuffles (MOV) and address
arithmetic the compiler leaves in the k loop.

usage: sass_loop.py file [function-substring]
"""
import collections
import re
import subprocess
import sys


def main():
    path = sys.argv[1]
    sub = sys.argv[2] if len(sys.argv) > 2 else ""
    txt = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    for part in re.split(r"\n\s+Function : ", txt)[1:]:
        name = part.split("\n")[0]
        if sub not in name:
            continue
        ins = []
        for m in re.finditer(r"/\*([0-9a-f]{4,5})\*/\s+(.*?);", part):
            ins.append((int(m.group(1), 16), m.group(2)))
        loops = []
        for i, (a, t) in enumerate(ins):
            m = re.search(r"BRA(?:\.\w+)*\s+(?:!?U?P\w+,\s*)?0x([0-9a-f]+)", t)
            if not m:
                continue
            tgt = int(m.group(1), 16)
            if tgt >= a:
                continue
            body = [x for y, x in ins if tgt <= y <= a]
            nf = sum(1 for x in body if re.search(r"\b(FFMA2|DMMA|FFMA)\b", x))
            loops.append((nf, body, tgt, a))
        if not loops or not max(l[0] for l in loops):
            continue
        # the innermost loop holding at least half of the busiest loop's FMAs
        top = max(l[0] for l in loops)
        best = min((l for l in loops if l[0] * 2 >= top), key=lambda l: len(l[1]))
        nf, body, tgt, a = best
        ops = collections.Counter((x.split()[1] if x.startswith("@") else x.split()[0]).split(".")[0] for x in body)
        other = len(body) - ops["FFMA2"] - ops["LDS"] - ops["MOV"]
        print("%-70s loop %05x-%05x: %d inst, FFMA2 %d, LDS %d, MOV %d, other %d (%.3f inst/FFMA2)"
              % (name[:70], tgt, a, len(body), ops["FFMA2"], ops["LDS"], ops["MOV"], other,
                 len(body) / max(1, ops["FFMA2"])))


if __name__ == "__main__":
    main()
