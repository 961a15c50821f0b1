"""Does CUDA context creation slow down when the process already holds a large
touched host heap? (dev helper; argv[1] = GB to touch first)"""
import ctypes
import sys
import time

import numpy as np

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0
t0 = time.perf_counter()
if gb > 0:
    a = np.ones(int(gb * 2**30) // 8)
t1 = time.perf_counter()
cudart = ctypes.CDLL("libcudart.so.12") if False else None
sys.path.insert(0, ".")
from paper_2305_14641_b200 import native as N  # noqa: E402
t2 = time.perf_counter()
N.device_count()
t3 = time.perf_counter()
off = np.array([0, 1, 2], np.int64)
g = N.Csr(off, np.array([1, 0], np.int32), None, 10.0)
N.cluster_sweep(g, [1.0])
t4 = time.perf_counter()
print(f"touch {gb} GB {t1 - t0:.2f}s  import {t2 - t1:.2f}s  cuInit {t3 - t2:.3f}s  first call {t4 - t3:.3f}s")
