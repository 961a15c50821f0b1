"""Potential time of small sigma batches (S = 1, 2, 4) on the bench graphs
(dev_potentials, CUDA events) and the host-API single-sigma cluster call
(dev helper). Prints one JSON line."""
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

graphgen.build()
res = {}
for wl, fn in (("lfr1m", graphgen.lfr), ("rmat22", graphgen.rmat)):
    off, nbr = fn()
    n = len(off) - 1
    csr = N.Csr(off, nbr, None, 10.0)
    dg = N.DeviceCsr(csr, torch.device("cuda", 0))
    st = torch.cuda.Stream()
    out = torch.empty((n, 4), dtype=torch.float64, device="cuda")
    r = {}
    for S in (1, 2, 4):
        sig = np.array([5.0, 2.0, 9.0, 20.0][:S])
        t = []
        for rep in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            N.dev_potentials(dg, sig, 0, n, out, st)
            e1.record(st)
            e1.synchronize()
            if rep:
                t.append(e0.elapsed_time(e1))
        r[f"potentials_S{S}_ms"] = statistics.median(t)
    w = []
    for rep in range(4):
        t0 = time.perf_counter()
        N.cluster(csr, 5.0)
        if rep:
            w.append(1e3 * (time.perf_counter() - t0))
    r["cluster_sigma5_host_api_ms"] = statistics.median(w)
    res[wl] = r
print(json.dumps(res))
