"""Small end-to-end exercise of every device entry point, for compute-sanitizer
(memcheck / racecheck / initcheck) runs on the GPU box. Exits non-zero on a
parity failure."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import pyoracle as O
from paper_2305_14641_b200 import native as N
from tests import helpers as H

def check(a, b):
    assert np.array_equal(np.asarray(a).view(np.int64), np.asarray(b).view(np.int64))

g, names, lab, k = H.karate()
sig = O.log_sigma_grid(10.0, 12)
res, v, succ = N.cluster_sweep(g.csr(N), sig, want_v=True, want_succ=True)
for q, s in enumerate(sig):
    check(v[q], O.potentials(g.offsets, g.nbr, g.wt, 10.0, s))
w = H.random_graph(301, 4.0, seed=3)            # weighted, odd N (tail column)
for mode in (N.EXP_EIGEN, N.EXP_GLIBC):
    N.set_exp_mode(mode)
    got = N.potentials(w.csr(N), [0.7, 2.3, 30.0])
    for q, s in enumerate([0.7, 2.3, 30.0]):
        check(got[q], O.potentials(w.offsets, w.nbr, w.wt, 10.0, s, mode=mode))
N.set_exp_mode(N.EXP_EIGEN)
N.set_kernel(N.KERNEL_REPLAY)
check(N.potentials(w.csr(N), sig), np.stack([O.potentials(w.offsets, w.nbr, w.wt, 10.0, s) for s in sig]))
N.set_kernel(N.KERNEL_FASTFWD)
hub = H.G(2001, np.zeros(1500, np.int32), np.arange(1, 1501, dtype=np.int32))
res, v, succ = N.cluster_sweep(hub.csr(N), sig, want_v=True, want_succ=True)
for q, s in enumerate(sig):
    vo, so, co, cio, ko = O.cluster(hub.offsets, hub.nbr, hub.wt, 10.0, s)
    check(v[q], vo); assert np.array_equal(succ[q], so) and np.array_equal(res[q].cluster_index, cio)
assert N.node_potential(w.csr(N), 5, 1.3) == O.potentials(w.offsets, w.nbr, w.wt, 10.0, 1.3)[5]
r = N.resolve_centers(np.array([1, 2, 3, 3, 3], np.int32)); assert r.num_clusters == 1
try:
    N.resolve_centers(np.array([1, 0, 7], np.int32)); raise SystemExit("expected cycle")
except N.LogicError:
    pass
dg = N.DeviceCsr(w.csr(N)); S = len(sig)
V = torch.empty((w.n, S), dtype=torch.float64, device="cuda"); N.dev_potentials(dg, sig, 0, w.n, V)
sc = torch.empty((w.n, S), dtype=torch.int32, device="cuda"); N.dev_successors(dg, V, S, 0, 150, sc[:150]); N.dev_successors(dg, V, S, 150, w.n, sc[150:])
c = torch.empty((S, w.n), dtype=torch.int32, device="cuda"); ci = torch.empty_like(c); nc = torch.empty(S, dtype=torch.int32, device="cuda")
ws = torch.empty(N.dev_resolve_workspace(w.n, S), dtype=torch.uint8, device="cuda")
N.dev_resolve(w.n, S, sc, c, ci, nc, ws); torch.cuda.synchronize()
# k-hop extension: hop cap 2 (on-chip sort + bitset emission: a row with > 512
# candidates) and 3 (expand + segmented sort), odd N
u = H.random_graph(1201, 9.0, seed=5, unit=True)
star_rows = np.arange(1, 700, dtype=np.int32)
kh = H.G(1201, np.concatenate([u.nbr[:0], np.zeros(699, np.int32)]), star_rows)
for gg in (u, kh):
    for K in (2, 3):
        N.set_hop_cap(K)
        got = N.potentials(gg.csr(N), [0.9, 6.0])
        for q, s in enumerate([0.9, 6.0]):
            check(got[q], O.potentials_khop(gg.offsets, gg.nbr, gg.wt, 10.0, s, K))
N.set_hop_cap(1)
print("sanitize smoke ok")
