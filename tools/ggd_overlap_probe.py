"""Does a concurrent device->host copy slow the GGD kernels? (dev helper)
Times dev_ggd on 16-sigma halves of the LFR field alone and while a 64 MB
pinned D2H runs on another stream."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench_tools import graphgen as G  # noqa: E402
from paper_2305_14641_b200 import native as N  # noqa: E402
from paper_2305_14641_b200.sweep import log_sigma_grid  # noqa: E402

o, nb = G.lfr()
n = len(o) - 1
g = N.Csr(o, nb, None, 10.0)
dg = N.DeviceCsr(g)
sig = np.array(log_sigma_grid(10.0, 32))
V = torch.empty((n, 32), dtype=torch.float64, device="cuda")
N.dev_potentials(dg, sig, 0, n, V)
half = [V[:, :16].contiguous(), V[:, 16:].contiguous()]
center = torch.empty((16, n), dtype=torch.int32, device="cuda")
ci = torch.empty_like(center)
nc = torch.empty(16, dtype=torch.int32, device="cuda")
ws = torch.empty(N.dev_ggd_workspace(n, 16), dtype=torch.uint8, device="cuda")
src = torch.empty(16 * n, dtype=torch.int32, device="cuda")
dst = torch.empty(16 * n, dtype=torch.int32).pin_memory()
cs = torch.cuda.Stream()
st = torch.cuda.Stream()


def ggd(h, copy):
    torch.cuda.synchronize()
    if copy:
        with torch.cuda.stream(cs):
            dst.copy_(src, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    N.dev_ggd(dg, half[h], 16, None, center, ci, nc, ws, st)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for rep in range(3):
    print("half0 alone %.3f  half1 alone %.3f  half0+copy %.3f  half1+copy %.3f" % (
        ggd(0, False), ggd(1, False), ggd(0, True), ggd(1, True)))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(cs)
with torch.cuda.stream(cs):
    dst.copy_(src, non_blocking=True)
e1.record(cs)
torch.cuda.synchronize()
print("64 MB D2H alone %.3f ms = %.1f GB/s" % (e0.elapsed_time(e1), 64e6 / e0.elapsed_time(e1) / 1e6))
