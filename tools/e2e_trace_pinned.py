import os, sys, time, statistics
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from bench_tools import graphgen
from paper_2305_14641_b200 import native as N
from paper_2305_14641_b200.sweep import log_sigma_grid
off, nbr = graphgen.lfr(); n = len(off) - 1
po, pn = torch.from_numpy(off).pin_memory().numpy(), torch.from_numpy(nbr).pin_memory().numpy()
sig = np.ascontiguousarray(log_sigma_grid(10.0, 32))
ci = torch.empty((32, n), dtype=torch.int32).pin_memory().numpy(); k = np.zeros(32, np.int32)
csr = N.Csr(po, pn, None, 10.0)
for rep in range(6):
    t0 = time.perf_counter(); N.cluster_sweep_raw(csr, sig, None, ci, k); print(f"wall {1e3*(time.perf_counter()-t0):.2f} ms", flush=True)
