"""A/B of the GGD chunk cuts of gqc_cluster_sweep (GQC_GGD_CUTS) on the bench
e2e call: LFR 1M x 32 sigmas, pinned host CSR and labels. One subprocess per
variant (the env is read per call, but keep processes clean)."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, time, statistics, json
sys.path.insert(0, %r)
import numpy as np, torch
from bench_tools import graphgen
from paper_2305_14641_b200 import native as N
from paper_2305_14641_b200.sweep import log_sigma_grid
off, nbr = getattr(graphgen, sys.argv[1])(); n = len(off) - 1
po, pn = torch.from_numpy(off).pin_memory().numpy(), torch.from_numpy(nbr).pin_memory().numpy()
sig = np.ascontiguousarray(log_sigma_grid(10.0, 32))
ci = torch.empty((32, n), dtype=torch.int32).pin_memory().numpy(); k = np.zeros(32, np.int32)
csr = N.Csr(po, pn, None, 10.0)
N.cluster_sweep_raw(csr, sig, None, ci, k)
ref = ci.copy()
ts = []
for rep in range(15):
    t0 = time.perf_counter(); N.cluster_sweep_raw(csr, sig, None, ci, k); ts.append(1e3 * (time.perf_counter() - t0))
assert np.array_equal(ci, ref)
print(json.dumps({"median_ms": statistics.median(ts), "min_ms": min(ts)}))
""" % ROOT

out = {}
for wl in sys.argv[1:] or ["lfr"]:
    for cuts in (os.environ["CUTS"].split(";") if os.environ.get("CUTS") else ["", "8,8,16", "4,8,8,12", "4,12,16", "8,24", "4,28", "16,8,8", "12,20"]):
        env = dict(os.environ)
        env.pop("GQC_GGD_CUTS", None)
        if cuts:
            env["GQC_GGD_CUTS"] = cuts
        r = subprocess.run([sys.executable, "-c", CHILD, wl], env=env, capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.returncode == 0 else r.stderr[-300:]
        out[f"{wl}:{cuts or 'default16'}"] = line
        print(wl, cuts or "default16", line, flush=True)
with open(os.path.join(ROOT, "gpurun_out", "e2e_cuts_ab.json"), "w") as f:
    json.dump(out, f, indent=1)
