"""Stage trace of the e2e call (gqc_cluster_sweep with pinned buffers) on the
bench workload: GQC_TRACE=1 prints CUDA-event stage times (dev helper)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_tools import graphgen  # noqa: E402
from paper_2305_14641_b200 import native as N  # noqa: E402
from paper_2305_14641_b200.sweep import log_sigma_grid  # noqa: E402

off, nbr = graphgen.lfr()
n, S = len(off) - 1, 32
pin_off = torch.from_numpy(off).pin_memory()
pin_nbr = torch.from_numpy(nbr).pin_memory()
csr = N.Csr(pin_off.numpy(), pin_nbr.numpy(), None, 10.0)
ci = torch.empty((S, n), dtype=torch.int32).pin_memory().numpy()
k = np.zeros(S, np.int32)
sig = np.ascontiguousarray(log_sigma_grid(10.0, S))
for it in range(6):
    t0 = time.perf_counter()
    N.cluster_sweep_raw(csr, sig, None, ci, k)
    print(f"call {it}: {1e3 * (time.perf_counter() - t0):.3f} ms", flush=True)
