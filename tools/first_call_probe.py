"""Per-process first-call costs of the C-ABI (what a CLI run pays once):
library load, CUDA init, first call (context + module load + pools), then
repeated LFR 1M calls at S=1 and S=30 with pageable numpy outputs, plus the
same calls through the facade CLI path. Prints one line per step (dev helper).
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("GQC_TRACE", "1")

t0 = time.perf_counter()


def lap(what, t=[t0]):
    now = time.perf_counter()
    print(f"{what:40s} {1e3 * (now - t[0]):9.1f} ms", flush=True)
    t[0] = now


import numpy as np  # noqa: E402

from bench_tools import graphgen as G  # noqa: E402
from paper_2305_14641_b200 import native  # noqa: E402

lap("imports")
native.lib()
lap("dlopen libgqc")
print("devices", native.device_count())
lap("device_count (cuInit)")
off = np.array([0, 1, 2], np.int64)
nbr = np.array([1, 0], np.int32)
g2 = native.Csr(off, nbr, None, 10.0)
native.cluster_sweep(g2, [1.0])
lap("first call, 2-node graph")
native.cluster_sweep(g2, [1.0])
lap("second call, 2-node graph")
o, nb = G.lfr()
g = native.Csr(o, nb, None, 10.0)
lap("generate LFR 1M")
for r in range(3):
    native.cluster_sweep(g, [5.0])
    lap(f"LFR S=1 call {r}")
grid = np.exp(np.linspace(np.log(1.0), np.log(30.0), 30))
for r in range(2):
    native.cluster_sweep(g, grid, want_center=False)
    lap(f"LFR S=30 call {r}")
