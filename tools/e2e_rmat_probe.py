"""gqc_cluster_sweep on R-MAT scale 22 x 32 sigmas with stage tracing (dev helper)."""
import os, sys, time
os.environ["GQC_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench_tools import graphgen
from paper_2305_14641_b200 import native as N
from paper_2305_14641_b200.sweep import log_sigma_grid
wl = sys.argv[1] if len(sys.argv) > 1 else "rmat"
off, nbr = graphgen.rmat() if wl == "rmat" else graphgen.lfr()
n = len(off) - 1
sig = np.array(log_sigma_grid(10.0, 32))
po, pn = torch.from_numpy(off).pin_memory(), torch.from_numpy(nbr).pin_memory()
csr = N.Csr(po.numpy(), pn.numpy(), None, 10.0)
ci = torch.empty((32, n), dtype=torch.int32).pin_memory().numpy()
k = np.zeros(32, np.int32)
for _ in range(3):
    t0 = time.perf_counter(); N.cluster_sweep_raw(csr, sig, None, ci, k); print(wl, "e2e ms", round((time.perf_counter() - t0) * 1e3, 2), flush=True)
