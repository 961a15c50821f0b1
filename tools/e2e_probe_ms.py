"""e2e of the bench workload through gqc_cluster_sweep with pinned host
buffers (ms per call, median of 10) for LFR 1M / R-MAT 22 / SBM 100k (dev helper)."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench_tools import graphgen  # noqa: E402
from paper_2305_14641_b200 import native as N  # noqa: E402
from paper_2305_14641_b200.sweep import log_sigma_grid  # noqa: E402

graphgen.build()
out = {}
for wl, fn in (("lfr1m", graphgen.lfr), ("sbm100k", graphgen.sbm), ("rmat22", graphgen.rmat)):
    off, nbr = fn()
    n = len(off) - 1
    po, pn = torch.from_numpy(off).pin_memory().numpy(), torch.from_numpy(nbr).pin_memory().numpy()
    sig = np.ascontiguousarray(log_sigma_grid(10.0, 32))
    ci = torch.empty((32, n), dtype=torch.int32).pin_memory().numpy()
    k = np.zeros(32, np.int32)
    csr = N.Csr(po, pn, None, 10.0)
    t = []
    for rep in range(12):
        t0 = time.perf_counter()
        N.cluster_sweep_raw(csr, sig, None, ci, k)
        if rep >= 2:
            t.append(1e3 * (time.perf_counter() - t0))
    out[wl] = round(statistics.median(t), 3)
print(json.dumps(out))
