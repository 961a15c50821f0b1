"""The multi-device sweep (gqc_cluster_sweep_multi / gqc_potentials_multi /
GQC_OPT_GPUS): the reference's compute_potentials_parallel row blocks
(potential.cpp:62-87) with GPUs as the workers, for cluster (ggd.cpp:59-62)
and run_sweep (sweep.cpp:50-57).

This environment gives one GPU, so the shard logic (cost-balanced row
blocks, sigma chunk ownership, the potential kernel's per-chunk output
pointers, cross-shard event ordering, per-shard GGD and label placement) runs
with several shards on device 0: `devices=[0] * k`. Every output must equal
the single-device sweep's bit for bit. No kernel waits on another here: the
shards are ordered by stream events only."""
import threading

import numpy as np
import pytest

from tests import helpers as H

pytestmark = pytest.mark.gpu

N = pytest.importorskip("paper_2305_14641_b200.native")


def same(a, b):
    if a is None or b is None:
        return a is None and b is None
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype == np.float64:
        return np.array_equal(a.view(np.int64), b.view(np.int64))
    return np.array_equal(a, b)


def check_multi(csr, sigmas, shards, intra=False):
    ref, v_ref, s_ref = N.cluster_sweep(csr, sigmas, want_v=True, want_succ=True)
    res, v, succ, it = N.cluster_sweep_multi(csr, sigmas, [0] * shards, want_v=True, want_succ=True,
                                             want_intra=intra)
    assert same(v, v_ref), f"{shards} shards: potentials differ"
    assert same(succ, s_ref), f"{shards} shards: successors differ"
    for q in range(len(sigmas)):
        assert same(res[q].center, ref[q].center) and same(res[q].cluster_index, ref[q].cluster_index)
        assert res[q].num_clusters == ref[q].num_clusters
    if intra:
        _, k1, it1 = N.cluster_sweep_intra(csr, sigmas)
        assert np.array_equal(it, it1)
    assert same(N.potentials_multi(csr, sigmas, [0] * shards), v_ref)


@pytest.mark.parametrize("shards", [2, 3, 8, 32])
def test_small_graphs_all_shard_counts(shards):
    from oracle import pyoracle as O
    grid = O.log_sigma_grid(10.0)
    g, _, _, _ = H.karate()
    check_multi(g.csr(N), grid, shards, intra=True)
    gw = H.random_graph(1001, 7, 5, unit=False)   # weighted, odd N (Eigen tail column)
    check_multi(gw.csr(N), grid[:9], shards)
    gu = H.random_graph(4000, 12, 6, unit=True)
    check_multi(gu.csr(N), np.concatenate([grid, [0.05, 300.0]]), shards, intra=True)


def test_more_shards_than_rows_and_sigmas():
    g = H.path(5)
    check_multi(g.csr(N), [2.0], 8)           # 1 sigma: shards 1..7 own no sigma; rows < shards
    check_multi(g.csr(N), [1.0, 2.0, 3.0], 4)
    g1 = H.star(0)                            # one node
    check_multi(g1.csr(N), [1.0, 5.0], 3)


def test_glibc_mode_and_replay_kernel():
    g = H.random_graph(777, 6, 8, unit=False)
    N.set_exp_mode(N.EXP_GLIBC)
    try:
        check_multi(g.csr(N), [0.5, 2.0, 7.0, 30.0], 3)
    finally:
        N.set_exp_mode(N.EXP_EIGEN)
    N.set_kernel(N.KERNEL_REPLAY)
    try:
        check_multi(H.random_graph(1500, 9, 9, unit=True).csr(N), [1.0, 2.2727, 5.0, 10.0, 30.0], 4)
    finally:
        N.set_kernel(N.KERNEL_FASTFWD)


def test_khop_extension_multi():
    g = H.random_graph(3000, 8, 10, unit=True)
    N.set_hop_cap(2)
    try:
        check_multi(g.csr(N), [1.0, 3.0, 8.0, 20.0, 30.0], 4)
    finally:
        N.set_hop_cap(1)


@pytest.mark.parametrize("workload", ["sbm100k", "lfr1m", "rmat22"])
def test_bench_graphs_eight_shards(workload):
    """8 shards of the bench graphs; on R-MAT the shards' launches walk hub rows
    (>= 1024 neighbours) whole (kLong) while the single-device launch uses the
    chunked walk, so this also pins the two walks to each other bit for bit."""
    from bench_tools import graphgen
    from paper_2305_14641_b200.sweep import log_sigma_grid
    graphgen.build()
    off, nbr = {"sbm100k": graphgen.sbm, "lfr1m": graphgen.lfr, "rmat22": graphgen.rmat}[workload]()
    check_multi(N.Csr(off, nbr, None, 10.0), np.asarray(log_sigma_grid(10.0, 32)), 8, intra=True)


def test_option_gpus_routes_host_entry_points():
    g = H.random_graph(2000, 10, 11, unit=True)
    csr = g.csr(N)
    sig = [1.0, 2.0, 5.0, 9.0, 12.0, 20.0, 25.0, 30.0]
    ref, v_ref, _ = N.cluster_sweep(csr, sig, want_v=True)
    assert N.get_gpus() == 1
    if N.device_count() < 2:
        with pytest.raises(ValueError, match="exceeds the visible devices"):
            N.set_gpus(2)
            try:
                N.cluster_sweep(csr, sig)
            finally:
                N.set_gpus(1)
    else:
        N.set_gpus(2)
        try:
            res, v, _ = N.cluster_sweep(csr, sig, want_v=True)
        finally:
            N.set_gpus(1)
        assert same(v, v_ref) and all(same(a.cluster_index, b.cluster_index) for a, b in zip(res, ref))
    with pytest.raises(ValueError):
        N.set_gpus(0)
    with pytest.raises(ValueError):
        N.cluster_sweep_multi(csr, sig, [0, 99])  # device ordinal out of range


def test_concurrent_calls_from_threads():
    """Per-device locks: calls from several host threads are serialized on
    one device and each gets its own results."""
    graphs = [H.random_graph(3000 + 100 * t, 9, 20 + t, unit=True) for t in range(4)]
    sig = [1.0, 2.0, 3.0, 5.0, 8.0, 13.0, 21.0, 30.0]
    want = [N.cluster_sweep(g.csr(N), sig, want_v=True)[1] for g in graphs]
    got = [None] * 4
    errs = []

    def work(t):
        try:
            for _ in range(3):
                got[t] = N.cluster_sweep_multi(graphs[t].csr(N), sig, [0] * (t + 1), want_v=True)[1]
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs
    assert all(same(a, b) for a, b in zip(got, want))
