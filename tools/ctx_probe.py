"""CUDA context creation cost on this box, without libgqc (dev helper):
cudaFree(0) through the runtime torch ships, then libgqc's gqc_init."""
import ctypes
import ctypes.util
import glob
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

import site  # noqa: E402

cands = []
for d in site.getsitepackages():
    cands += glob.glob(os.path.join(d, "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
rt = ctypes.CDLL(cands[0])
t0 = time.perf_counter()
rt.cudaFree(None)
t1 = time.perf_counter()
sys.path.insert(0, ROOT)
from paper_2305_14641_b200 import native as N  # noqa: E402
t2 = time.perf_counter()
N.lib().gqc_init()
t3 = time.perf_counter()
print(f"cudart context {1e3 * (t1 - t0):.0f} ms, import libgqc {1e3 * (t2 - t1):.0f} ms, "
      f"gqc_init (own runtime: context + pool + module load + tiny sweep) {1e3 * (t3 - t2):.0f} ms, "
      f"CUDA_MODULE_LOADING={os.environ.get('CUDA_MODULE_LOADING', 'default')}")
