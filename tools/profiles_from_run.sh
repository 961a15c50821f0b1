#!/bin/bash
# Refresh profiles/ from the gpurun_out/ artefacts of tools/gpu_profile_r02.sh
# (here, after the run): traffic.json, metric extracts, launch list, K2 source.
set -e
cd "$(dirname "$0")/.."
echo '{}' > profiles/traffic.json
for w in lfr1m sbm100k rmat22; do
  python tools/traffic_from_ncu.py gpurun_out/r02_full_$w.ncu-rep $w \
    --source "r02 final pass: ncu --set full --clock-control none, python bench.py --profile --steps 1 --warmup 1 --workload $w (32 sigmas)" > /dev/null
done
python tools/traffic_from_ncu.py gpurun_out/r02_full_replay_sbm100k.ncu-rep sbm100k > /dev/null
python - <<'PY'
import csv, json, os, subprocess, collections
keep = ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed", "smsp__cycles_elapsed.avg",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__warps_eligible.avg.per_cycle_active", "launch__grid_size", "launch__block_size",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct")
for name, rep in (("lfr1m", "r02_full_lfr1m"), ("sbm100k", "r02_full_sbm100k"), ("rmat22", "r02_full_rmat22"),
                  ("sbm100k_replay", "r02_full_replay_sbm100k")):
    out = subprocess.run(["ncu", "-i", f"gpurun_out/{rep}.ncu-rep", "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    cols = [i for i, x in enumerate(h) if x in keep]
    with open(f"profiles/r02_ncu_{name}.csv", "w", newline="") as f:
        csv.writer(f).writerows([[h[i] for i in cols], [u[i] for i in cols]] + [[r[i] for i in cols] for r in rows[2:]])
t = json.load(open("profiles/traffic.json"))
for wl, d in t["workloads"].items():
    for k, v in d.items():
        if isinstance(v, dict) and "report" in v:
            base = os.path.basename(v["report"])
            v["report"] = ("profiles/r02_ncu_sbm100k_replay.csv" if "replay" in base else f"profiles/r02_ncu_{wl}.csv") \
                + f" (from {base}, ncu --set full)"
json.dump(t, open("profiles/traffic.json", "w"), indent=1, sort_keys=True)
rows = list(csv.reader(open("gpurun_out/launches.csv")))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]; ki, vi = h.index("Kernel Name"), h.index("Metric Value")
out = ["# ncu launch list (gpu__time_duration.sum, --clock-control none), `python bench.py --profile --steps 1 --warmup 1` (LFR 1M, 32 sigmas), r02 final pass: warm-up step + timed step",
       "# cold-cache, serialized per launch: compare SHARES, not absolute step times", "kernel,duration_ns"]
per = collections.OrderedDict(); tot = 0.0
for r in rows[hi + 1:]:
    nm = r[ki].split("(")[0].replace("void ", "").replace("gqc::<unnamed>::", "")
    v = float(r[vi].replace(",", "")); out.append(f"{nm},{v:.0f}"); per[nm] = per.get(nm, 0) + v; tot += v
out.append(f"# total {tot:.0f} ns")
for k, v in sorted(per.items(), key=lambda x: -x[1]):
    out.append(f"# share {k[:60]}: {100 * v / tot:.1f}%")
open("profiles/r02_launches.csv", "w").write("\n".join(out) + "\n")
PY
(echo "# ncu --set full, LFR 1M x 32 sigmas, r02 final pass: details of the two captured kernels, then the top source lines of both (warp instructions executed, stall-sample share)"; python tools/ncu_summary.py gpurun_out/r02_full_lfr1m.ncu-rep 30) > profiles/r02_ncu_lfr1m_source.txt 2>&1
