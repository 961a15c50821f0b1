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
# multi-device sweep (3 shards on device 0: per-chunk output pointers, event
# ordering, per-shard GGD) and the device CSR build
ref, v1, _ = N.cluster_sweep(u.csr(N), sig, want_v=True)
got, v2, _, _ = N.cluster_sweep_multi(u.csr(N), sig, [0, 0, 0], want_v=True, want_intra=True)
check(v1, v2)
assert all(np.array_equal(a.cluster_index, b.cluster_index) for a, b in zip(ref, got))
rng = np.random.default_rng(1)
eu, ev = rng.integers(0, 500, 4000).astype(np.int32), rng.integers(0, 500, 4000).astype(np.int32)
off, nbr, wt, unit, dups = N.build_csr(500, eu, ev, rng.choice([1.0, 2.0], 4000))
ro, rn, rw = O.csr_from_edges(500, eu, ev, None, 10.0)
assert np.array_equal(off, ro) and np.array_equal(nbr, rn)
# bounded chase + pointer jumping on a 5000-node monotone chain (dev_ggd)
pth = H.path(5000)
dp = N.DeviceCsr(pth.csr(N))
ar = torch.arange(5000, dtype=torch.float64, device="cuda")
Vp = torch.stack([5000.0 - ar, ar], dim=1).contiguous()
sp = torch.empty((2, 5000), dtype=torch.int32, device="cuda"); cp = torch.empty_like(sp); cip = torch.empty_like(sp)
ncp = torch.empty(2, dtype=torch.int32, device="cuda")
wsp = torch.empty(N.dev_ggd_workspace(5000, 2), dtype=torch.uint8, device="cuda")
N.dev_ggd(dp, Vp, 2, sp, cp, cip, ncp, wsp); torch.cuda.synchronize()
assert list(ncp.cpu().numpy()) == [1, 1] and int(cp[0, 0]) == 4999 and int(cp[1, 4999]) == 0
# polled CSR upload (>= 2^20 entries, 8 sigmas): flags released by a kernel
big = H.random_graph(110_000, 20.0, seed=9, unit=True)
assert big.offsets[-1] >= (1 << 20)
res_b, vb, _ = N.cluster_sweep(big.csr(N), sig[:8], want_v=True)
rows = np.arange(0, big.n, 9973, dtype=np.int32)
for q, s in enumerate(sig[:8]):
    check(vb[q][rows], O.potentials_rows(big.offsets, big.nbr, big.wt, 10.0, s, rows, workers=8))
print("sanitize smoke ok")
