"""GPU parity of the opt-in k-hop distance extension (GQC_OPT_HOP_CAP > 1,
khop.cu; not a reference feature) against its CPU oracle
(oracle.cpp fill_khop, itself checked against the definition and, at K = 1,
against the reference's distance in test_oracle.py). Bit for bit, like the
K = 1 path: the BFS events, the exact fast-forward and the GGD labels."""
import os

import numpy as np
import pytest

from oracle import pyoracle as O
from tests import helpers as H

pytestmark = pytest.mark.gpu

N = pytest.importorskip("paper_2305_14641_b200.native")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
SIG = np.array([0.05, 0.5, 1.0, 2.0, 3.0, 5.0, 8.0, 12.0, 20.0, 30.0])


@pytest.fixture(autouse=True)
def _reset():
    yield
    N.set_hop_cap(1)
    N.set_exp_mode(N.EXP_EIGEN)


def assert_bits(a, b):
    a, b = np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64)
    bad = np.flatnonzero(a.view(np.int64) != b.view(np.int64))
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:5]}: {a.ravel()[bad[:5]]} vs {b.ravel()[bad[:5]]}"


def full_check(g, K, sigmas=SIG, mode=N.EXP_EIGEN):
    N.set_exp_mode(mode)
    N.set_hop_cap(K)
    res, v, succ = N.cluster_sweep(g.csr(N), sigmas, want_v=True, want_succ=True)
    for q, s in enumerate(sigmas):
        ref = O.potentials_khop(g.offsets, g.nbr, g.wt, g.W, s, K, workers=4, mode=mode)
        assert_bits(v[q], ref)
        so = O.build_successors(g.offsets, g.nbr, ref)
        assert np.array_equal(succ[q], so)
        co, cio, ko = O.resolve_centers(so)
        assert np.array_equal(res[q].center, co) and np.array_equal(res[q].cluster_index, cio)
        assert res[q].num_clusters == ko


@pytest.mark.parametrize("K", [2, 3, 4, 7])
@pytest.mark.parametrize("n,deg,seed", [(301, 6, 1), (400, 3, 2), (1001, 12, 3), (64, 1, 4)])
def test_random_graphs_khop_bitwise(K, n, deg, seed):
    full_check(H.random_graph(n, deg, seed, unit=True), K)


@pytest.mark.parametrize("fname", ["karate.edges", "les_miserables.edges", "florentine.edges", "davis.edges",
                                   "planted_4x32.edges"])
@pytest.mark.parametrize("K", [2, 3])
def test_small_graphs_khop_bitwise(fname, K):
    g, _ = H.parse_edge_list(os.path.join(GOLDEN, fname))
    if not g.unit:
        pytest.skip("weighted")
    full_check(g, K)


def test_khop_glibc_mode_and_structured_graphs():
    full_check(H.star(40), 2, mode=N.EXP_GLIBC)
    full_check(H.path(33), 5)
    full_check(H.complete(9), 2)
    full_check(H.planted(4, 25, 0.3, 0.02, 5), 3, mode=N.EXP_GLIBC)


def test_khop_one_is_the_reference_distance():
    g = H.random_graph(500, 7, 8, unit=True)
    N.set_hop_cap(1)
    a = N.potentials(g.csr(N), SIG)
    N.set_hop_cap(2)
    b = N.potentials(g.csr(N), SIG)
    N.set_hop_cap(1)
    c = N.potentials(g.csr(N), SIG)
    assert_bits(a, c)
    for q, s in enumerate(SIG):
        assert_bits(a[q], O.potentials(g.offsets, g.nbr, g.wt, g.W, s, workers=4))
    assert not np.array_equal(a, b)


def test_khop_weighted_graph_rejected():
    g = H.random_graph(50, 4, 9, unit=False)
    N.set_hop_cap(2)
    with pytest.raises(ValueError, match="k-hop distances need unit weights"):
        N.potentials(g.csr(N), [1.0])
    with pytest.raises(ValueError, match="k-hop distances need unit weights"):
        N.cluster_sweep(g.csr(N), [1.0])


def test_khop_node_potential_and_single_sigma():
    g = H.random_graph(777, 9, 10, unit=True)
    N.set_hop_cap(3)
    for i in (0, 1, 388, 776):
        got = N.node_potential(g.csr(N), i, 2.2727)
        ref = O.potentials_khop(g.offsets, g.nbr, g.wt, g.W, 2.2727, 3, rows=[i])
        assert_bits([got], ref)
    one = N.potentials(g.csr(N), [4.0])
    assert_bits(one[0], O.potentials_khop(g.offsets, g.nbr, g.wt, g.W, 4.0, 3, workers=4))


def test_khop_sbm_100k_sampled_rows():
    off, nbr = H.sbm_csr()
    csr = N.Csr(off, nbr, None, 10.0)
    sig = np.array([1.0, 2.2727, 5.0, 30.0])
    N.set_hop_cap(2)
    v = N.potentials(csr, sig)
    rows = np.arange(0, csr.n, 3001, dtype=np.int32)
    for q, s in enumerate(sig):
        assert_bits(v[q][rows], O.potentials_khop(off, nbr, None, 10.0, s, 2, workers=8, rows=rows))


def test_khop_global_bitset_path_large_n():
    # N above the shared-memory bitset limit (1.6M bits): global-memory bitsets
    n = 1_700_001
    rng = np.random.default_rng(11)
    u = rng.integers(0, n, 3 * n // 2).astype(np.int32)
    v = rng.integers(0, n, 3 * n // 2).astype(np.int32)
    g = H.G(n, u, v)
    N.set_hop_cap(2)
    got = N.potentials(g.csr(N), [3.0, 9.0])
    rows = np.array([0, 1, 17, n // 2, n - 2, n - 1], dtype=np.int32)
    for q, s in enumerate([3.0, 9.0]):
        assert_bits(got[q][rows], O.potentials_khop(g.offsets, g.nbr, g.wt, g.W, s, 2, workers=6, rows=rows))


def test_khop_device_row_shards_assemble():
    torch = pytest.importorskip("torch")
    g = H.random_graph(2001, 10, 12, unit=True)
    N.set_hop_cap(2)
    full = N.potentials(g.csr(N), SIG[:8])
    dg = N.DeviceCsr(g.csr(N))
    out = torch.empty((g.n, 8), dtype=torch.float64, device="cuda")
    for b, e in [(0, 700), (700, 1500), (1500, g.n)]:
        N.dev_potentials(dg, SIG[:8], b, e, out[b:e])
    torch.cuda.synchronize()
    assert_bits(out.cpu().numpy().T, full)
