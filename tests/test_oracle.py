"""Pins the CPU oracle (oracle/oracle.cpp) to every golden vector and known
answer the reference publishes for this path. CPU only."""
import math

import numpy as np
import pytest

from oracle import pyoracle as O
from tests import helpers as H

README_ROW = ("0.3122945430637738,0.6486360381182862,0.6684671059738576,0.8319365867687499,"
              "0.9032258064516129,0.9117647058823529,0.8235294117647058,2,5")  # proj/README.md:58-59
README_MUTATION = "mutation interval: [2.272723014236749, 2.5555343651620004] drop=17\n"  # proj/README.md:69
MODES = [O.EXP_EIGEN, O.EXP_GLIBC]


@pytest.mark.parametrize("mode", MODES)
def test_karate_report_row_golden(mode):
    a, r = O.run_cluster(H.KARATE_EDGES, H.KARATE_LABELS, 5.0, workers=2, mode=mode)
    assert r == "modularity,nmi,ari,fmi,f1,accuracy,recall,num_clusters,sigma\n" + README_ROW + "\n"
    rows = a.strip().split("\n")
    assert rows[0] == "node,center,cluster" and len(rows) == 35
    assert len({r.rsplit(",", 1)[1] for r in rows[1:]}) == 2


@pytest.mark.parametrize("mode", MODES)
def test_karate_default_sweep_mutation_golden(mode):
    s, m = O.run_sweep(H.KARATE_EDGES, H.KARATE_LABELS, mode=mode)
    assert m == README_MUTATION
    assert s.startswith("sigma,num_clusters,modularity,nmi,ari,fmi\n")


def test_karate_centers_golden():
    # ggd_test.cpp:144-156: sigma=5, W=10 -> centers "0" and "33", 14 nodes in cluster 0
    g, names, lab, k = H.karate()
    v, succ, center, ci, nc = O.cluster(g.offsets, g.nbr, g.wt, 10.0, 5.0, workers=2)
    assert nc == 2
    centers = sorted(set(center.tolist()))
    assert [names[c] for c in centers] == ["0", "33"]
    assert int((ci == 0).sum()) == 14


def test_karate_shape():
    # graph_test.cpp:165-178
    g, names, lab, k = H.karate()
    assert g.n == 34 and len(g.nbr) == 2 * 78
    deg = np.diff(g.offsets)
    assert deg[names.index("0")] == 16 and deg[names.index("33")] == 17
    assert k == 2 and (lab == 0).sum() == 17


def test_karate_linear_plateau_two_clusters():
    # sweep_test.cpp:144-153
    s, m = O.run_sweep(H.KARATE_EDGES, None, sigma_min=10.0, sigma_max=300.0, steps=30, log_grid=False, workers=2)
    counts = [int(line.split(",")[1]) for line in s.strip().split("\n")[1:]]
    assert counts == [2] * 30
    assert m == "mutation interval: none\n"


@pytest.mark.parametrize("mode", MODES)
def test_star_tiny_sigma(mode):
    # sweep_test.cpp:72-89
    g = H.star(8)
    _, _, center, _, nc = O.cluster(g.offsets, g.nbr, g.wt, 10.0, 0.2, mode=mode)
    assert nc == 8 and all(center[leaf] == leaf for leaf in range(1, 9))
    _, _, center, _, nc = O.cluster(g.offsets, g.nbr, g.wt, 10.0, 0.01, mode=mode)
    assert nc == 1 and center[0] == 0


def test_single_node_and_two_node_closed_form():
    # potential_test.cpp:26-41
    g = H.G(1, np.zeros(0, np.int32), np.zeros(0, np.int32))
    assert O.potentials(g.offsets, g.nbr, g.wt, 10.0, 1.0)[0] == 0.0
    d, sigma = 2.5, 1.3
    g = H.G(2, np.array([0]), np.array([1]), np.array([d]))
    e = math.exp(-d * d / (2 * sigma * sigma))
    expected = d * d / (2 * sigma * sigma) * e / (1 + e)
    v = O.potentials(g.offsets, g.nbr, g.wt, 10.0, sigma)
    assert all(abs(x - expected) / expected < 1e-12 for x in v)


def test_star_orderings():
    # potential_test.cpp:43-61
    g = H.star(4)
    v = O.potentials(g.offsets, g.nbr, g.wt, 10.0, 5.0)
    assert all(v[0] < v[leaf] for leaf in range(1, 5))
    v = O.potentials(g.offsets, g.nbr, g.wt, 10.0, 1.0)
    assert all(v[0] > v[leaf] for leaf in range(1, 5))


def test_ggd_small_goldens():
    # ggd_test.cpp:41-57, :92-101
    g = H.path(3)
    succ = O.build_successors(g.offsets, g.nbr, np.array([3.0, 1.0, 2.0]))
    assert succ.tolist() == [1, 1, 1]
    center, ci, k = O.resolve_centers(succ)
    assert k == 1 and center.tolist() == [1, 1, 1] and ci.tolist() == [0, 0, 0]
    g = H.G(2, np.array([0]), np.array([1]))
    assert O.build_successors(g.offsets, g.nbr, np.array([0.7, 0.7])).tolist() == [0, 0]
    tri = H.G(6, np.array([0, 1, 0, 3, 4, 3]), np.array([1, 2, 2, 4, 5, 5]))
    _, _, center, ci, k = O.cluster(tri.offsets, tri.nbr, tri.wt, 10.0, 1.0)
    assert k == 2 and ci.tolist() == [0, 0, 0, 1, 1, 1]
    with pytest.raises(RuntimeError, match="cycle"):
        O.resolve_centers(np.array([1, 0]))
    with pytest.raises(ValueError, match="out of range"):
        O.resolve_centers(np.array([5, 0]))
    center, ci, k = O.resolve_centers(np.array([1, 2, 3, 3, 3]))
    assert k == 1 and center.tolist() == [3] * 5


def test_metric_goldens():
    # metrics_test.cpp:65-97, cli_test.cpp:192-194
    s = O.scores([0, 0, 1, 1], 2, [0, 0, 0, 1], 2)
    assert s["ari"] == 0.0
    assert s["fmi"] == 1.0 / math.sqrt(6.0)
    assert O.scores([0, 0, 1, 1], 2, [1, 1, 0, 0], 2)["ari"] == 1.0
    assert O.scores([0, 1, 2], 3, [2, 1, 0], 3)["ari"] == 1.0
    assert O.scores([0, 1, 2], 3, [0, 0, 0], 1)["ari"] == 0.0
    assert O.scores([0, 1, 0, 1], 2, [0, 0, 0, 0], 1)["nmi"] == 0.0


def test_sigma_grids():
    # sweep_test.cpp:23-39
    g = O.log_sigma_grid(10.0)
    assert len(g) == 30 and abs(g[0] - 1.0) < 1e-12 and abs(g[-1] - 30.0) < 1e-9
    assert O.linear_sigma_grid(2.0, 4.0, 5).tolist() == [2.0, 2.5, 3.0, 3.5, 4.0]
    assert O.detect_mutation([1, 2, 3, 4], [10, 9, 3, 2]) == (2.0, 3.0, 6)
    assert O.detect_mutation([1, 2, 3, 4], [8, 5, 5, 2]) == (1.0, 2.0, 3)
    assert O.detect_mutation([1, 2, 3], [5, 5, 5]) is None


def test_pexp_restatement_properties():
    # exp(0) == 1 exactly (the self term), the survey's subnormal clamp, and
    # agreement with glibc to 1 ulp on the exp arguments this path uses.
    assert O.eigen_pexp(0.0) == 1.0 and O.eigen_pexp(-0.0) == 1.0
    assert O.eigen_pexp(-5000.0) == pytest.approx(5.55552948377339e-309, rel=1e-12)
    rng = np.random.default_rng(0)
    for x in -rng.random(2000) * 700.0:
        a, b = O.eigen_pexp(x), O.glibc_exp(x)
        assert abs(a - b) <= 2 * np.spacing(b)


def test_parallel_equals_serial_bitwise():
    # potential_test.cpp:92-103
    for n in (3, 37, 256):
        g = H.random_graph(n, 4.0, seed=303 + n)
        serial = O.potentials(g.offsets, g.nbr, g.wt, 10.0, 1.7, workers=1)
        for w in (2, 4, 8):
            assert np.array_equal(O.potentials(g.offsets, g.nbr, g.wt, 10.0, 1.7, workers=w), serial)


def test_oracle_vs_definition():
    # potential_test.cpp:69-78: the field matches the definition (std::exp) to 1e-12
    for trial in range(4):
        g = H.random_graph(60, 4.0, seed=101 + trial)
        sigma = 0.7 if trial % 2 == 0 else 6.0
        v = O.potentials(g.offsets, g.nbr, g.wt, 10.0, sigma)
        for i in range(g.n):
            d = np.full(g.n, 10.0)
            d[g.nbr[g.offsets[i]:g.offsets[i + 1]]] = g.wt[g.offsets[i]:g.offsets[i + 1]]
            d[i] = 0.0
            d2 = d * d
            e = np.exp(-d2 / (2 * sigma * sigma))
            ref = (d2 * e).sum() / e.sum() / (2 * sigma * sigma)
            assert abs(v[i] - ref) <= 1e-12 * max(abs(ref), 1e-300)


def test_khop_oracle_matches_definition_and_reference_distance():
    """k-hop extension (oracle.cpp fill_khop): hop_cap 1 is the reference's
    distance bit for bit; hop_cap K matches a direct restatement of the
    definition (networkx BFS hop counts, W beyond K, the Eigen packet / glibc
    tail exp rule, ascending fp64 sums) on small graphs."""
    import networkx as nx
    for n, deg, seed in [(41, 3, 1), (40, 2, 2), (57, 5, 3)]:
        g = H.random_graph(n, deg, seed, unit=True)
        for sigma in (0.7, 2.0, 6.0):
            base = O.potentials(g.offsets, g.nbr, g.wt, g.W, sigma)
            k1 = O.potentials_khop(g.offsets, g.nbr, g.wt, g.W, sigma, 1)
            assert np.array_equal(base.view(np.int64), k1.view(np.int64))
        G = nx.Graph()
        G.add_nodes_from(range(n))
        for i in range(n):
            for k in range(g.offsets[i], g.offsets[i + 1]):
                G.add_edge(i, int(g.nbr[k]))
        for K in (2, 3, 5):
            got = O.potentials_khop(g.offsets, g.nbr, g.wt, g.W, 2.5, K, workers=2)
            inv = 1.0 / (2.0 * 2.5 * 2.5)
            for i in range(n):
                hops = nx.single_source_shortest_path_length(G, i, cutoff=K)
                d2 = [float(hops[j]) ** 2 if j in hops else g.W * g.W for j in range(n)]
                ex = [O.eigen_pexp(-inv * x) if j < n - n % 2 else O.glibc_exp(-inv * x) for j, x in enumerate(d2)]
                num = den = 0.0
                for x, e in zip(d2, ex):
                    num += x * e
                    den += e
                assert got[i] == inv * (num / den)
    with pytest.raises(ValueError, match="k-hop distances need unit weights"):
        w = H.random_graph(30, 3, 9, unit=False)
        O.potentials_khop(w.offsets, w.nbr, w.wt, w.W, 1.0, 2)
