#!/usr/bin/env python3
"""Summarise `ncu --set full` captures (.ncu-rep) into the text/JSON kept
under profiles/ (the .ncu-rep files themselves stay in gpurun_out/).

    python tools/ncu_summary.py NAME=path.ncu-rep [...] --out profiles/ncu_rNN.json
        [--traffic profiles/traffic.json]

NAME is the bench shape name (e.g. f32_NN_80x80x80); --traffic merges
dram__bytes_read.sum + dram__bytes_write.sum per launch into the file bench.py
reads for the roofline "traffic" field.
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__inst_executed.sum", "smsp__sass_inst_executed_op_shared_ld.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "smsp__sass_inst_executed_op_local_ld.sum",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
    "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
]
STALLS = "smsp__average_warps_issue_stalled_%s_per_issue_active.ratio"


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for i, h in enumerate(hdr):
            d[h] = (r[i], units[i])
        res.append(d)
    return res


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return v


def scale(v, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
    return v * mult[unit] if isinstance(v, float) and unit in mult else v


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="+")
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic")
    a = ap.parse_args()
    summary = {}
    for spec in a.reps:
        name, path = spec.split("=", 1)
        for d in raw(path):
            s = {"kernel": d["Kernel Name"][0], "rep": path.split("/")[-1]}
            for k in KEYS:
                if k in d:
                    s[k] = scale(num(d[k][0]), d[k][1])
                    if d[k][1] and d[k][1] not in ("byte", "Kbyte", "Mbyte", "Gbyte", "ns", "us", "ms"):
                        s[k + " [unit]"] = d[k][1]
            st = {}
            for k, (v, _) in d.items():
                if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                    st[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = num(v)
            s["stalls_per_issue"] = dict(sorted(((k, v) for k, v in st.items() if isinstance(v, float) and v >= 0.01),
                                                key=lambda kv: -kv[1]))
            summary[name] = s
    with open(a.out, "w") as f:
        json.dump(summary, f, indent=1)
    if a.traffic:
        try:
            with open(a.traffic) as f:
                t = json.load(f)
        except FileNotFoundError:
            t = {}
        for name, s in summary.items():
            t[name] = s["dram__bytes_read.sum"] + s["dram__bytes_write.sum"]
        with open(a.traffic, "w") as f:
            json.dump(t, f, indent=1, sort_keys=True)
    for name, s in summary.items():
        print("%-20s %-30s t=%.1fus dram=%.1fMB fma=%.1f%% issue=%.1f%% smem_wf=%.1f%%" % (
            name, s["kernel"][:30], s["gpu__time_duration.sum"] * 1e6,
            (s["dram__bytes_read.sum"] + s["dram__bytes_write.sum"]) / 1e6,
            s.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 0),
            s.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0),
            s.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 0)))


if __name__ == "__main__":
    main()
