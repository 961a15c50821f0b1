"""Time the reference-facing C-ABI sweep (gqc_cluster_sweep) on LFR 1M x 32
sigmas with pinned host buffers (dev helper for the e2e leg of bench.py)."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench_tools import graphgen
from paper_2305_14641_b200 import native as N
from paper_2305_14641_b200.sweep import log_sigma_grid
off, nbr = graphgen.lfr()
n = len(off) - 1
sig = np.array(log_sigma_grid(10.0, 32))
po, pn = torch.from_numpy(off).pin_memory(), torch.from_numpy(nbr).pin_memory()
csr = N.Csr(po.numpy(), pn.numpy(), None, 10.0)
ci = torch.empty((32, n), dtype=torch.int32).pin_memory().numpy()
k = np.zeros(32, np.int32)
N.cluster_sweep_raw(csr, sig, None, ci, k)
ts = []
for _ in range(8):
    t0 = time.perf_counter(); N.cluster_sweep_raw(csr, sig, None, ci, k); ts.append(time.perf_counter() - t0)
print("e2e ms", round(statistics.mean(ts) * 1e3, 3), "min", round(min(ts) * 1e3, 3))
