#!/usr/bin/env python3
"""Reduced cases of every kernel family, for compute-sanitizer:
    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_cases.py
Each case is checked against the oracle after the run; exit 0 when all pass."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def force(**kw):
    for k in list(os.environ):
        if k.startswith("IAAT_FORCE_"):
            os.environ.pop(k)
    for k, v in kw.items():
        os.environ["IAAT_FORCE_" + k.upper()] = str(v)


def main():
    import torch
    from tests.gpu_utils import Case, CCase
    F32, F64 = np.float32, np.float64
    cases = [
        ("slab fp32 NN (bulk copy)", dict(family=0), (F32, "N", "N", 24, 20, 17, 37, 1.5, 0.5, {})),
        ("slab fp32 TN odd ld (scalar)", dict(family=0), (F32, "T", "N", 13, 11, 7, 29, 1.0, 0.25, {"pad": 1})),
        ("slab fp64 DMMA", dict(family=1), (F64, "N", "T", 16, 24, 12, 21, 1.0, 0.0, {})),
        ("ks TMA fp32 TT", dict(family=2), (F32, "T", "T", 36, 28, 44, 23, 1.5, 0.5, {"ld_multiple": 4})),
        ("ks LDGSTS fp32 NN odd ld", dict(family=2), (F32, "N", "N", 21, 19, 33, 17, 1.0, 1.0, {"pad": 1})),
        ("ks DMMA fp64 NN", dict(family=3), (F64, "N", "N", 32, 40, 36, 19, 1.0, 0.5, {})),
        ("ksg fp32 NN", dict(family=7), (F32, "N", "N", 48, 48, 40, 41, 1.5, 0.5, {})),
        ("ksg fp32 TT padded", dict(family=7), (F32, "T", "T", 44, 52, 37, 19, 1.5, 0.0, {"ld_multiple": 4})),
    ]
    ok = True
    for name, kn, (dt, ta, tb, M, N, K, batch, al, be, extra) in cases:
        force(**kn)
        c = Case(dt, ta, tb, M, N, K, batch, 3, al, be, **extra)
        c.run()
        torch.cuda.synchronize()
        err, _, _ = c.check()
        print("%-32s err %.2e" % (name, err), flush=True)
    force()
    cc = CCase(np.complex128, "N", "T", 16, 16, 16, 13, 2, 0.5 - 1j, 1j)
    cc.run()
    torch.cuda.synchronize()
    print("%-32s err %.2e" % ("ZGEMM DMMA NT", cc.check()), flush=True)
    cc = CCase(np.complex64, "T", "N", 9, 7, 5, 13, 2, 0.5 - 1j, 1j)
    cc.run()
    torch.cuda.synchronize()
    print("%-32s err %.2e" % ("CGEMM slab TN", cc.check()), flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
