#!/usr/bin/env python3
"""FLOP and DRAM audit of single launches from ncu counters.

On the GPU box (one ncu run per case, one launch each):
    python tools/audit.py run OUTDIR
Here (no GPU), from the CSVs it wrote:
    python tools/audit.py summarise OUTDIR profiles/audit_r01.json

Per launch: FMA thread-instructions (FFMA + 2*FFMA2, or 256*DMMA + DFMA)
against M*N*K*batch + the epilogue's one FMA per C element when beta != 0
(exact tiles: no padded or predicated work), and DRAM bytes read against
the algorithmic input bytes (M*K + K*N + [beta != 0]*M*N) * elt * batch (no
pack pass, no re-reads).  DRAM writes are reported but not audited: ncu
stops counting with part of C still dirty in the 126 MB L2.
"""
import csv
import json
import os
import subprocess
import sys

CASES = [  # dtype, trans, M, N, K, batch, alpha, beta
    ("f32", "NN", 64, 64, 64, 5461, 1.5, 0.5),
    ("f32", "TT", 68, 68, 68, 4837, 1.5, 0.5),
    ("f32", "NT", 80, 80, 80, 3495, 1.5, 0.5),
    ("f32", "NN", 37, 67, 79, 100000, 1.0, 1.0),
    ("f32", "TN", 29, 29, 29, 500000, -1.0, 0.25),
    ("f32", "NN", 16, 16, 16, 87381, 1.5, 0.0),
    ("f64", "NN", 64, 64, 64, 200000, 1.0, 0.0),
    ("f64", "NT", 80, 80, 80, 100000, 1.0, 0.0),
]
METRICS = ("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum,"
           "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__inst_executed_pipe_tensor_subpipe_dmma.sum,"
           "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum")


def name(c):
    return "%s_%s_%dx%dx%d_b%d_beta%g" % (c[0], c[1], c[2], c[3], c[4], c[5], c[7])


def run(out):
    os.makedirs(out, exist_ok=True)
    for c in CASES:
        cmd = ["ncu", "--metrics", METRICS, "--clock-control", "none", "-k", "regex:iaat", "-s", "3", "-c", "1",
               "--csv", "--log-file", os.path.join(out, name(c) + ".csv"), sys.executable, "tools/run_case.py",
               c[0], c[1], str(c[2]), str(c[3]), str(c[4]), str(c[5]), "--alpha", str(c[6]), "--beta", str(c[7])]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
        print(name(c), r.returncode, flush=True)


def summarise(out, dst):
    res = {}
    for c in CASES:
        p = os.path.join(out, name(c) + ".csv")
        if not os.path.exists(p):
            continue
        vals, kern = {}, None
        for row in csv.reader(open(p)):
            if len(row) > 14 and row[0] not in ("ID", "") and row[-3] in METRICS.split(","):
                vals[row[-3]] = float(row[-1].replace(",", ""))
                kern = row[4]
        if not vals:
            continue
        dt, tr, M, N, K, batch, alpha, beta = c
        elt = 4 if dt == "f32" else 8
        fma = (vals.get("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", 0) +
               2 * vals.get("smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum", 0) +
               vals.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0) +
               256 * vals.get("smsp__inst_executed_pipe_tensor_subpipe_dmma.sum", 0))
        want = M * N * K * batch + (M * N * batch if beta != 0 else 0)
        rd_alg = (M * K + K * N + (M * N if beta != 0 else 0)) * elt * batch
        res[name(c)] = {"kernel": kern, "fma_thread_inst": fma, "expected": want, "fma_ratio": fma / want,
                        "dram_read": vals.get("dram__bytes_read.sum"), "dram_read_alg": rd_alg,
                        "read_ratio": vals.get("dram__bytes_read.sum", 0) / rd_alg,
                        "dram_write": vals.get("dram__bytes_write.sum"), "write_alg": M * N * elt * batch,
                        "metrics": vals}
    json.dump(res, open(dst, "w"), indent=1)
    for k, v in res.items():
        print("%-40s fma %.6f read %.4f  %s" % (k, v["fma_ratio"], v["read_ratio"], v["kernel"][:40]))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        summarise(sys.argv[2], sys.argv[3])
