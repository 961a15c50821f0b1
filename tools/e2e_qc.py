"""End-to-end QC time through the graphqc CLI (load edge list
-> CSR -> potentials -> GGD -> metrics -> outputs, graphqc_main.cpp:92-157).

Writes the LFR-style 1M graph (bench_tools/graphgen, seed 1) and its planted
communities as text files, then times `graphqc sweep` (default 30-point log
grid) and `graphqc cluster --sigma 5` with GQC_TRACE=1 stage timings. Each
command runs `--repeat` times; the first run includes CUDA context creation.
Prints one JSON line. Usage (GPU box):
    python tools/e2e_qc.py [--n 1000000] [--dir /tmp/e2e_qc] [--repeat 2]
"""
import argparse
import json
import os
import re
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench_tools import graphgen as G  # noqa: E402

CLI = os.path.join(ROOT, "paper_2305_14641_b200", "bin", "graphqc")


def stages(stderr):
    return {m.group(1): float(m.group(2)) for m in re.finditer(r"\[graphqc\] (\w+)\s+([\d.]+) ms", stderr)}


def run(cmd, repeat):
    out = []
    for _ in range(repeat):
        t0 = time.perf_counter()
        p = subprocess.run(cmd, capture_output=True, text=True, env=dict(os.environ, GQC_TRACE="1"))
        wall = time.perf_counter() - t0
        if p.returncode != 0:
            raise SystemExit(f"{cmd} failed ({p.returncode}): {p.stderr[-2000:]}")
        trace = [l for l in p.stderr.splitlines()
                 if l.startswith("[gqc trace]") or "sweep:" in l or "load:" in l or "device init" in l]
        out.append({"wall_s": round(wall, 3), "stages_ms": stages(p.stderr), "trace": trace,
                    "stdout_tail": p.stdout[-200:]})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--dir", default="/tmp/e2e_qc")
    ap.add_argument("--repeat", type=int, default=2)
    a = ap.parse_args()
    os.makedirs(a.dir, exist_ok=True)
    edges, labels = os.path.join(a.dir, "lfr.edges"), os.path.join(a.dir, "lfr.labels")
    t0 = time.perf_counter()
    off, nbr = G.lfr(a.n)
    lab = G.labels(a.n)
    G.write_edge_list(edges, off, nbr)
    with open(labels, "w") as f:
        f.write("\n".join(f"{i} {c}" for i, c in enumerate(lab.tolist())))
        f.write("\n")
    gen = time.perf_counter() - t0
    res = {"workload": f"LFR-style N={a.n}, nnz {len(nbr)}, unit weights, planted communities as labels",
           "edge_file_bytes": os.path.getsize(edges), "gen_s": round(gen, 2), "host_threads": os.cpu_count()}
    res["sweep"] = run([CLI, "sweep", edges, "--labels", labels, "--out", os.path.join(a.dir, "sweep.csv")],
                       a.repeat)
    res["cluster_sigma5"] = run([CLI, "cluster", edges, "--labels", labels, "--sigma", "5",
                                 "--out", os.path.join(a.dir, "assign.csv")], a.repeat)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
