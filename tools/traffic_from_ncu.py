"""Update profiles/traffic.json from an `ncu --set full` report (dev helper).

    python tools/traffic_from_ncu.py REPORT.ncu-rep WORKLOAD [--source "..."]

For every kernel launch in the report (the last launch of each kernel name
wins) it records, per launch, dram bytes read/written, duration, warp
instructions, issue-slot utilisation, active threads per warp, FP64 pipe
utilisation and registers, under workloads[WORKLOAD][kernel key]. bench.py
attaches these figures only to the bench line of the same workload.
"""
import argparse
import csv
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
FIELDS = {
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "duration_ms": "gpu__time_duration.sum",
    "inst_executed": "smsp__inst_executed.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "threads_per_warp": "smsp__thread_inst_executed_per_inst_executed.ratio",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dadd_per_cycle": "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed",
    "cycles_elapsed": "smsp__cycles_elapsed.avg",
}


def kernel_key(name):
    m = re.search(r"(\w+)<([^>]*)>\s*\(", name)
    if m and m.group(1) == "potential_warp_kernel":
        args = [a.strip() for a in m.group(2).split(",")]
        ff, w = args[0], args[1]
        key = f"potential_warp_kernel<{'FASTFWD' if ff == '1' else 'REPLAY'},{ {'0': 'unit', '1': 'pexp', '2': 'table'}[w] }"
        return key + (",long>" if len(args) > 2 and args[2] in ("1", "true") else ">")
    m = re.search(r"(\w+)(<[^(]*>)?\s*\(", name)
    return m.group(1) if m else name


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("workload")
    ap.add_argument("--source", default="")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    res = {}
    for r in rows[2:]:
        key = kernel_key(r[col["Kernel Name"]])
        d = {}
        for f, m in FIELDS.items():
            if m not in col:
                continue
            try:
                v = float(r[col[m]].replace(",", ""))
            except ValueError:
                continue
            d[f] = v * SCALE.get(units[col[m]], 1.0)
        if "dadd_per_cycle" in d and "cycles_elapsed" in d:  # fp64 adds executed (thread level)
            d["dadd_thread_inst"] = d["dadd_per_cycle"] * d["cycles_elapsed"]
        if "dram_read" in d and "dram_write" in d:
            d["dram_bytes"] = d["dram_read"] + d["dram_write"]
        d["report"] = os.path.relpath(a.report, ROOT)
        res[key] = d
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        t = json.load(open(p))
    except (OSError, ValueError):
        t = {}
    t.setdefault("_source", "ncu --set full --clock-control none; per-launch figures; dram bytes = "
                            "dram__bytes_read.sum + dram__bytes_write.sum")
    t.setdefault("workloads", {}).setdefault(a.workload, {}).update(res)
    if a.source:
        t["workloads"][a.workload]["_source"] = a.source
    json.dump(t, open(p, "w"), indent=1, sort_keys=True)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
