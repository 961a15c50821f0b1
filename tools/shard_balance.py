"""Per-shard potential time of the multi-device row partition (gqc_row_shards)
on ONE GPU: each shard's row block is timed alone with gqc_dev_potentials
(CUDA events, 32 sigmas), so max/mean is the load imbalance the partition
would show across GPUs. Also times the reference's equal blocks
(potential.cpp:70-74) for comparison. Prints one JSON line.

    python tools/shard_balance.py [--workload rmat22|lfr1m|sbm100k] [--shards 8]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="rmat22")
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch

    from bench_tools import graphgen
    from paper_2305_14641_b200 import native as N
    from paper_2305_14641_b200.sweep import log_sigma_grid
    graphgen.build()
    off, nbr = {"rmat22": graphgen.rmat, "lfr1m": graphgen.lfr, "sbm100k": graphgen.sbm}[a.workload]()
    n = len(off) - 1
    sig = np.asarray(log_sigma_grid(10.0, 32))
    csr = N.Csr(off, nbr, None, 10.0)
    dev = torch.device("cuda", 0)
    dg = N.DeviceCsr(csr, dev)
    stream = torch.cuda.Stream(dev)
    out = torch.empty((n, 32), dtype=torch.float64, device=dev)
    k = a.shards
    balanced = [int(x) for x in N.row_shards(csr, k)]
    equal = [w * (n // k) + min(w, n % k) for w in range(k)] + [n]
    res = {"workload": a.workload, "n": n, "nnz": int(len(nbr)), "shards": k}
    for name, b in (("cost_balanced", balanced), ("equal_rows", equal)):
        times = []
        for r in range(k):
            t = []
            for rep in range(a.reps + 1):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                N.dev_potentials(dg, sig, b[r], b[r + 1], out[b[r]:], stream)
                e1.record(stream)
                e1.synchronize()
                if rep:
                    t.append(e0.elapsed_time(e1))
            times.append(statistics.median(t))
        res[name] = {"bounds": b, "ms": [round(x, 4) for x in times],
                     "max_over_mean": max(times) / statistics.mean(times),
                     "nnz": [int(off[b[r + 1]] - off[b[r]]) for r in range(k)]}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    N.dev_potentials(dg, sig, 0, n, out, stream)
    e1.record(stream)
    e1.synchronize()
    res["whole_ms"] = e0.elapsed_time(e1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
