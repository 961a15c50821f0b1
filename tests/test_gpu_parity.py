"""GPU parity: the sm_100a path, called through the C-ABI (libgqc.so), against
the CPU oracle on the same seeded inputs. Integer outputs (successors,
centers, cluster indices, counts) and the fp64 potentials are compared BIT
FOR BIT: the reference's labels on unit-weight graphs depend on the last bit
of the ascending-j sums, so the only tolerance is zero."""
import numpy as np
import pytest

from oracle import pyoracle as O
from tests import helpers as H

pytestmark = pytest.mark.gpu

N = pytest.importorskip("paper_2305_14641_b200.native")

KERNELS = [N.KERNEL_FASTFWD, N.KERNEL_REPLAY]
MODES = [N.EXP_EIGEN, N.EXP_GLIBC]


@pytest.fixture(autouse=True)
def _reset():
    yield
    N.set_exp_mode(N.EXP_EIGEN)
    N.set_kernel(N.KERNEL_FASTFWD)


def setup(kernel, mode):
    N.set_kernel(kernel)
    N.set_exp_mode(mode)


def oracle_field(g, sigma, mode):
    return O.potentials(g.offsets, g.nbr, g.wt, g.W, sigma, workers=4, mode=mode)


def assert_bits(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape
    bad = np.flatnonzero(a.view(np.int64) != b.view(np.int64))
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:5]}: {a.ravel()[bad[:5]]} vs {b.ravel()[bad[:5]]}"


SIGMAS = [0.05, 0.3, 1.0, 1.7, 2.3, 5.0, 30.0, 500.0]


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("mode", MODES)
def test_karate_potentials_bitwise(kernel, mode):
    setup(kernel, mode)
    g, names, lab, k = H.karate()
    grid = O.log_sigma_grid(10.0)
    sig = np.concatenate([grid, SIGMAS])
    sig.sort()
    got = N.potentials(g.csr(N), sig)
    for q, s in enumerate(sig):
        assert_bits(got[q], oracle_field(g, s, mode))


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("n", [2, 3, 37, 200, 257])
@pytest.mark.parametrize("unit", [True, False])
def test_random_graph_potentials_bitwise(kernel, mode, n, unit):
    # oracles::random_graph shapes (odd and even N: the Eigen tail column)
    setup(kernel, mode)
    g = H.random_graph(n, 4.0, seed=1000 + n, unit=unit)
    got = N.potentials(g.csr(N), SIGMAS)
    for q, s in enumerate(SIGMAS):
        assert_bits(got[q], oracle_field(g, s, mode))


@pytest.mark.parametrize("kernel", KERNELS)
def test_structured_graphs_bitwise(kernel):
    # stars, paths, complete graphs (long coalesced neighbour runs), planted partitions
    setup(kernel, N.EXP_EIGEN)
    graphs = [H.star(8), H.star(9), H.path(50), H.path(51), H.complete(33), H.complete(64),
              H.planted(4, 32, 0.3, 0.02, seed=1), H.planted(5, 31, 0.3, 0.02, seed=2)]
    for g in graphs:
        got = N.potentials(g.csr(N), SIGMAS)
        for q, s in enumerate(SIGMAS):
            assert_bits(got[q], oracle_field(g, s, N.EXP_EIGEN))


def test_weights_stored_as_ones_equal_unit():
    g = H.random_graph(101, 5.0, seed=5, unit=True)
    a = N.potentials(g.csr(N, unit_as_null=False), SIGMAS)
    b = N.potentials(g.csr(N, unit_as_null=True), SIGMAS)
    assert_bits(a, b)


@pytest.mark.parametrize("mode", MODES)
def test_fastfwd_equals_replay_medium(mode):
    # N=4001 unit SBM-like graph, many sigmas including the underflow regime
    g = H.random_graph(4001, 16.0, seed=77, unit=True)
    sig = np.array(sorted(set(O.log_sigma_grid(10.0, 32).tolist() + [0.05, 0.2, 0.5])))
    N.set_exp_mode(mode)
    N.set_kernel(N.KERNEL_REPLAY)
    a = N.potentials(g.csr(N), sig)
    N.set_kernel(N.KERNEL_FASTFWD)
    b = N.potentials(g.csr(N), sig)
    assert_bits(a, b)
    rows = np.arange(0, g.n, 97, dtype=np.int32)
    for q in (0, 7, 15, 31):
        ref = O.potentials_rows(g.offsets, g.nbr, g.wt, g.W, sig[q], rows, workers=8, mode=mode)
        assert_bits(b[q][rows], ref)


def test_sbm_100k_fastfwd_vs_replay_and_sampled_oracle():
    off, nbr = H.sbm_csr()
    csr = N.Csr(off, nbr, None, 10.0)
    sig = np.array([1.0, 2.2727, 5.0, 30.0])
    N.set_kernel(N.KERNEL_FASTFWD)
    b = N.potentials(csr, sig)
    N.set_kernel(N.KERNEL_REPLAY)
    a = N.potentials(csr, sig)
    assert_bits(a, b)
    rows = np.arange(0, csr.n, 1999, dtype=np.int32)
    for q, s in enumerate(sig):
        ref = O.potentials_rows(off, nbr, None, 10.0, s, rows, workers=8)
        assert_bits(b[q][rows], ref)


@pytest.mark.parametrize("kernel", KERNELS)
def test_node_potential_and_errors(kernel):
    setup(kernel, N.EXP_EIGEN)
    g = H.random_graph(31, 4.0, seed=9)
    full = N.compute_potentials(g.csr(N), 1.3)
    for i in (0, 15, 30):
        assert N.node_potential(g.csr(N), i, 1.3) == full[i]
    with pytest.raises(ValueError, match="sigma must be positive"):
        N.node_potential(g.csr(N), 0, 0.0)
    with pytest.raises(ValueError, match="sigma must be positive"):
        N.compute_potentials(g.csr(N), -2.0)
    with pytest.raises(ValueError, match="workers must be at least 1"):
        N.compute_potentials_parallel(g.csr(N), 1.0, 0)
    with pytest.raises(IndexError, match="out of range"):
        N.node_potential(g.csr(N), 31, 1.0)


def test_single_node_graph():
    g = H.G(1, np.zeros(0, np.int32), np.zeros(0, np.int32))
    assert N.node_potential(g.csr(N), 0, 1.0) == 0.0
    res = N.cluster(g.csr(N), 1.0)
    assert res.num_clusters == 1 and res.center.tolist() == [0]


@pytest.mark.parametrize("mode", MODES)
def test_karate_labels_and_report(mode):
    setup(N.KERNEL_FASTFWD, mode)
    g, names, lab, k = H.karate()
    res = N.cluster(g.csr(N), 5.0)
    assert res.num_clusters == 2
    assert [names[c] for c in res.centers] == ["0", "33"]
    row = O.metric_row(g.offsets, g.nbr, g.wt, 10.0, res.cluster_index, res.num_clusters, lab, k, 1.0, 5.0)
    assert row == ("0.3122945430637738,0.6486360381182862,0.6684671059738576,0.8319365867687499,"
                   "0.9032258064516129,0.9117647058823529,0.8235294117647058,2,5")


@pytest.mark.parametrize("mode", MODES)
def test_karate_sweep_mutation(mode):
    setup(N.KERNEL_FASTFWD, mode)
    g, names, lab, k = H.karate()
    grid = O.log_sigma_grid(10.0)
    res, v, succ = N.cluster_sweep(g.csr(N), grid, want_v=True, want_succ=True)
    counts = [r.num_clusters for r in res]
    assert O.detect_mutation(grid, counts) == (2.272723014236749, 2.5555343651620004, 17)
    for q, s in enumerate(grid):
        vo, so, co, cio, ko = O.cluster(g.offsets, g.nbr, g.wt, 10.0, s, mode=mode)
        assert_bits(v[q], vo)
        assert np.array_equal(succ[q], so) and np.array_equal(res[q].center, co)
        assert np.array_equal(res[q].cluster_index, cio) and res[q].num_clusters == ko


@pytest.mark.parametrize("unit", [True, False])
def test_cluster_sweep_random_graphs_labels(unit):
    for n in (40, 301, 1000):
        g = H.random_graph(n, 3.0, seed=45 + n, unit=unit)
        sig = O.log_sigma_grid(10.0, 12)
        res, v, succ = N.cluster_sweep(g.csr(N), sig, want_v=True, want_succ=True)
        for q, s in enumerate(sig):
            vo, so, co, cio, ko = O.cluster(g.offsets, g.nbr, g.wt, 10.0, s)
            assert_bits(v[q], vo)
            assert np.array_equal(succ[q], so)
            assert np.array_equal(res[q].center, co) and np.array_equal(res[q].cluster_index, cio)
            assert res[q].num_clusters == ko


def test_build_successors_and_resolve_on_random_potentials():
    # ggd_test.cpp:103-142 / acceptance criterion 4 (seed 45): random potentials
    rng = np.random.default_rng(45)
    for trial in range(20):
        n = int(rng.integers(2, 300))
        g = H.random_graph(n, 3.0, seed=trial)
        v = rng.random(n)
        if trial % 3 == 0:
            v = np.round(v * 4) / 4  # exact ties -> smaller id
        succ = N.build_successors(g.csr(N), v)
        assert np.array_equal(succ, O.build_successors(g.offsets, g.nbr, v))
        res = N.resolve_centers(succ)
        co, cio, ko = O.resolve_centers(succ)
        assert np.array_equal(res.center, co) and np.array_equal(res.cluster_index, cio) and res.num_clusters == ko


def test_resolve_centers_errors_match_reference_order():
    with pytest.raises(N.LogicError, match="successor map contains a cycle"):
        N.resolve_centers(np.array([1, 0], np.int32))
    with pytest.raises(ValueError, match="successor id out of range"):
        N.resolve_centers(np.array([5, 0], np.int32))
    # node 0 reaches a cycle before node 2 reaches an out-of-range id -> cycle
    with pytest.raises(N.LogicError):
        N.resolve_centers(np.array([1, 0, 7], np.int32))
    # node 0 reaches the out-of-range id first
    with pytest.raises(ValueError):
        N.resolve_centers(np.array([2, 1, -1, 4, 3], np.int32))
    res = N.resolve_centers(np.array([1, 2, 3, 3, 3], np.int32))
    assert res.num_clusters == 1 and res.center.tolist() == [3] * 5
    res = N.resolve_centers(np.array([0, 1, 2, 3], np.int32))
    assert res.num_clusters == 4
    with pytest.raises(ValueError, match="does not match graph size"):
        N.build_successors(H.path(3).csr(N), np.array([1.0, 2.0]))


def test_deep_chain_resolve():
    # long successor chains (a path with monotone potentials) stay O(N log N)
    n = 200_000
    succ = np.maximum(np.arange(n, dtype=np.int32) - 1, 0)
    res = N.resolve_centers(succ)
    assert res.num_clusters == 1 and (res.center == 0).all()
    g = H.path(5001)
    v = np.arange(g.n, dtype=np.float64)
    res = N.resolve_centers(N.build_successors(g.csr(N), v))
    assert res.num_clusters == 1


def test_tiny_sigma_star_fragments_and_collapses():
    # sweep_test.cpp:72-89 (the underflow tie case)
    g = H.star(8)
    res = N.cluster(g.csr(N), 0.2)
    assert res.num_clusters == 8 and all(res.center[l] == l for l in range(1, 9))
    res = N.cluster(g.csr(N), 0.01)
    assert res.num_clusters == 1 and res.centers.tolist() == [0]


def test_device_api_row_shards_assemble_to_full_field():
    import torch
    g = H.random_graph(5003, 8.0, seed=3, unit=True)
    dg = N.DeviceCsr(g.csr(N))
    sig = O.log_sigma_grid(10.0, 32)
    full = torch.empty((g.n, len(sig)), dtype=torch.float64, device="cuda")
    N.dev_potentials(dg, sig, 0, g.n, full)
    parts = []
    bounds = [0, 1000, 1001, 3333, 5003]
    for a, b in zip(bounds[:-1], bounds[1:]):
        t = torch.empty((b - a, len(sig)), dtype=torch.float64, device="cuda")
        N.dev_potentials(dg, sig, a, b, t)
        parts.append(t)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts).view(torch.int64), full.view(torch.int64))
    host = N.potentials(g.csr(N), sig)
    assert_bits(full.cpu().numpy().T.copy(), host)
    S = len(sig)
    succ = torch.empty((S, g.n), dtype=torch.int32, device="cuda")
    center = torch.empty_like(succ)
    ci = torch.empty_like(succ)
    nc = torch.empty(S, dtype=torch.int32, device="cuda")
    ws = torch.empty(N.dev_ggd_workspace(g.n, S), dtype=torch.uint8, device="cuda")
    N.dev_ggd(dg, full, S, succ, center, ci, nc, ws)
    torch.cuda.synchronize()
    res, _, s_host = N.cluster_sweep(g.csr(N), sig, want_succ=True)
    assert np.array_equal(succ.cpu().numpy(), s_host)
    assert np.array_equal(center.cpu().numpy(), np.stack([r.center for r in res]))
    assert nc.cpu().tolist() == [r.num_clusters for r in res]


@pytest.mark.parametrize("S,chunk", [(32, 32), (32, 8), (32, 4), (13, 5), (9, 1), (40, 7)])
@pytest.mark.parametrize("unit", [True, False])
def test_packed_potentials_are_a_rearrangement(S, chunk, unit):
    # gqc_dev_potentials_packed: sigma k of row i at (k // chunk) * stride +
    # (i - begin) * chunk + k % chunk, bit-identical to the node-major field;
    # padding slots of the last chunk are untouched
    import torch
    g = H.random_graph(3001, 6.0, seed=5, unit=unit)
    dg = N.DeviceCsr(g.csr(N))
    sig = O.log_sigma_grid(10.0, S)
    b, e = 1000, 2500
    full = torch.empty((e - b, S), dtype=torch.float64, device="cuda")
    N.dev_potentials(dg, sig, b, e, full)
    q = (S + chunk - 1) // chunk
    stride = (e - b) * chunk + 3
    packed = torch.full((q * stride,), -7.0, dtype=torch.float64, device="cuda")
    N.dev_potentials_packed(dg, sig, b, e, packed, chunk, stride)
    torch.cuda.synchronize()
    f, p = full.cpu().numpy(), packed.cpu().numpy()
    for k in range(q):
        blk = p[k * stride: k * stride + (e - b) * chunk].reshape(e - b, chunk)
        real = min(chunk, S - k * chunk)
        assert np.array_equal(blk[:, :real].view(np.int64), f[:, k * chunk: k * chunk + real].view(np.int64))
        assert np.all(blk[:, real:] == -7.0)
        assert np.all(p[k * stride + (e - b) * chunk: (k + 1) * stride] == -7.0)
    with pytest.raises(ValueError):
        N.dev_potentials_packed(dg, sig, b, e, packed, 0, stride)


def test_sigma_sharded_schedule_single_gpu_matches_cluster_sweep():
    # SigmaShardedSweep at world 1 (the bench schedule) through the device API
    import torch
    from paper_2305_14641_b200 import sharded
    g = H.random_graph(4000, 7.0, seed=8, unit=True)
    csr = g.csr(N)
    dg = N.DeviceCsr(csr)
    sig = O.log_sigma_grid(10.0, 32)
    S = len(sig)
    center = torch.empty((S, g.n), dtype=torch.int32, device="cuda")
    ws = torch.empty(N.dev_ggd_workspace(g.n, S), dtype=torch.uint8, device="cuda")
    sweep = sharded.SigmaShardedSweep(
        g.n, S, 0, 1, "cuda",
        lambda b, e, send, ch, st: N.dev_potentials_packed(dg, sig, b, e, send, ch, st),
        lambda v, ci, nc: N.dev_ggd(dg, v, S, None, center, ci, nc, ws))
    ci, nc = sweep.step()
    torch.cuda.synchronize()
    res, _, _ = N.cluster_sweep(csr, sig)
    assert np.array_equal(ci.cpu().numpy(), np.stack([r.cluster_index for r in res]))
    assert nc.cpu().tolist() == [r.num_clusters for r in res]


def _dev_labels(g_csr, sig):
    import torch
    dg = N.DeviceCsr(g_csr)
    S = len(sig)
    v = torch.empty((g_csr.n, S), dtype=torch.float64, device="cuda")
    N.dev_potentials(dg, sig, 0, g_csr.n, v)
    succ = torch.empty((S, g_csr.n), dtype=torch.int32, device="cuda")
    center, ci = torch.empty_like(succ), torch.empty_like(succ)
    nc = torch.empty(S, dtype=torch.int32, device="cuda")
    ws = torch.empty(N.dev_ggd_workspace(g_csr.n, S), dtype=torch.uint8, device="cuda")
    N.dev_ggd(dg, v, S, succ, center, ci, nc, ws)
    torch.cuda.synchronize()
    return v.cpu().numpy().T.copy(), succ.cpu().numpy(), center.cpu().numpy(), ci.cpu().numpy(), nc.cpu().numpy()


def test_pipelined_sweep_matches_device_path_sbm():
    # >= 2^20 nnz: the host API uploads the CSR in 4 row slabs under the
    # potential launches and downloads labels per 16-sigma chunk
    off, nbr = H.sbm_csr()
    csr = N.Csr(off, nbr, None, 10.0)
    sig = O.log_sigma_grid(10.0, 32)
    res, v, succ = N.cluster_sweep(csr, sig, want_v=True, want_succ=True)
    vd, sd, cd, cid, ncd = _dev_labels(csr, sig)
    assert_bits(v, vd)
    assert np.array_equal(succ, sd)
    assert np.array_equal(np.stack([r.center for r in res]), cd)
    assert np.array_equal(np.stack([r.cluster_index for r in res]), cid)
    assert [r.num_clusters for r in res] == ncd.tolist()
    res2, _, _ = N.cluster_sweep(csr, sig, want_center=False)
    assert np.array_equal(np.stack([r.cluster_index for r in res2]), cid)
    assert [r.num_clusters for r in res2] == ncd.tolist()


def test_pipelined_sweep_weighted_odd_n_sampled_oracle():
    # weighted, odd N (Eigen tail column), > 2^20 entries: slabbed weights upload
    n = 150_001
    g = H.random_graph(n, 8.0, seed=21)
    csr = g.csr(N)
    sig = np.array([0.7, 2.3, 5.0, 11.0, 30.0])
    res, v, succ = N.cluster_sweep(csr, sig, want_v=True, want_succ=True)
    rows = np.arange(0, n, 1499, dtype=np.int32)
    # plus every row adjacent to the tail column N-1 and the tail row itself
    rows = np.unique(np.concatenate([rows, g.nbr[g.offsets[n - 1]:g.offsets[n]], [n - 1]])).astype(np.int32)
    for q, s in enumerate(sig):
        ref = O.potentials_rows(g.offsets, g.nbr, g.wt, 10.0, s, rows, workers=8)
        assert_bits(v[q][rows], ref)
    vd, sd, cd, cid, ncd = _dev_labels(csr, sig)
    assert_bits(v, vd)
    assert np.array_equal(np.stack([r.cluster_index for r in res]), cid)


def test_hub_rows_heavy_argmin_and_scheduling():
    # hubs above the heavy-row threshold (kHeavyDegree = 256) take the
    # block-parallel argmin and the longest-first row schedule; everything
    # still matches the oracle
    rng = np.random.default_rng(11)
    n = 6001
    u = [np.zeros(3000, np.int32), np.full(1500, 17, np.int32), rng.integers(0, n, 6000).astype(np.int32)]
    v = [np.arange(1, 3001, dtype=np.int32), rng.choice(n, 1500, replace=False).astype(np.int32),
         rng.integers(0, n, 6000).astype(np.int32)]
    g = H.G(n, np.concatenate(u), np.concatenate(v))
    sig = O.log_sigma_grid(10.0, 12)
    res, V, succ = N.cluster_sweep(g.csr(N), sig, want_v=True, want_succ=True)
    for q, s in enumerate(sig):
        vo, so, co, cio, ko = O.cluster(g.offsets, g.nbr, g.wt, 10.0, s, workers=8)
        assert_bits(V[q], vo)
        assert np.array_equal(succ[q], so) and np.array_equal(res[q].cluster_index, cio) and res[q].num_clusters == ko
    # single-sigma path (thread-per-row potential kernel) and build_successors
    for s in (1.0, 5.0):
        vo = O.potentials(g.offsets, g.nbr, g.wt, 10.0, s, workers=8)
        assert np.array_equal(N.build_successors(g.csr(N), vo), O.build_successors(g.offsets, g.nbr, vo))


def test_row_sharded_successors_and_resolve_match_full_ggd():
    # the multi-GPU schedule's device pieces: successors of row shards
    # (node-major) assemble to the full argmin, and resolve() reproduces
    # dev_ggd's centers / labels / counts
    import torch
    from paper_2305_14641_b200 import sharded
    g = H.random_graph(5003, 8.0, seed=31, unit=True)
    csr = g.csr(N)
    sig = O.log_sigma_grid(10.0, 32)
    S = len(sig)
    v_ref, s_ref, c_ref, ci_ref, nc_ref = _dev_labels(csr, sig)
    dg = N.DeviceCsr(csr)
    center = torch.empty((S, g.n), dtype=torch.int32, device="cuda")
    ci, nc = torch.empty_like(center), torch.empty(S, dtype=torch.int32, device="cuda")
    ws = torch.empty(N.dev_resolve_workspace(g.n, S), dtype=torch.uint8, device="cuda")
    for world in (1, 3):
        V = torch.empty((g.n, S), dtype=torch.float64, device="cuda")
        N.dev_potentials(dg, sig, 0, g.n, V)
        succ = torch.empty((g.n, S), dtype=torch.int32, device="cuda")
        for r in range(world):
            b, e = sharded.row_shard(g.n, world, r)
            N.dev_successors(dg, V, S, b, e, succ[b:e])
        N.dev_resolve(g.n, S, succ, center, ci, nc, ws)
        torch.cuda.synchronize()
        assert np.array_equal(succ.cpu().numpy().T, s_ref)
        assert np.array_equal(center.cpu().numpy(), c_ref) and np.array_equal(ci.cpu().numpy(), ci_ref)
        assert nc.cpu().tolist() == nc_ref.tolist()


def hub_graph(n, seed):
    """Random sparse graph plus hub rows of degree 64..2000 (the batched walk):
    hubs at columns 0 and n-1 and in the middle, hubs adjacent to n-1 (the
    Eigen tail column when n is odd), neighbour lists spanning many 32-chunks."""
    rng = np.random.default_rng(seed)
    u, v, _ = H.graphgen.random_edges(n, 4.0, unit=True, seed=seed)
    us, vs = [u], [v]
    hubs = [0, n - 1, n // 2, n // 3 + 1, 7]
    for h, deg in zip(hubs, [300, 2000, 64, 65, 1000]):
        nb = rng.choice(n, size=min(deg, n - 1), replace=False)
        nb = nb[nb != h]
        us.append(np.full(len(nb), h, np.int32))
        vs.append(nb.astype(np.int32))
    # a hub whose neighbours are exactly the columns right below and above it
    h = n // 4
    nb = np.array([c for c in range(h - 40, h + 60) if c != h and 0 <= c < n], np.int32)
    us.append(np.full(len(nb), h, np.int32))
    vs.append(nb)
    return H.G(n, np.concatenate(us), np.concatenate(vs), None, 10.0)


@pytest.mark.parametrize("n", [4001, 4000])
def test_batched_walk_hub_rows_bitwise(n):
    # rows with >= 64 neighbours take the batched in-binade walk; every row of
    # every sigma (incl. tiny and huge) must equal the oracle and the replay
    g = hub_graph(n, seed=n)
    assert np.diff(g.offsets).max() >= 1000
    sig = sorted(set(list(O.log_sigma_grid(10.0, 32)) + [0.05, 0.3, 500.0]))
    field = N.potentials(g.csr(N), sig)
    for q, s in enumerate(sig):
        assert_bits(field[q], oracle_field(g, s, N.EXP_EIGEN))
    N.set_kernel(N.KERNEL_REPLAY)
    assert_bits(N.potentials(g.csr(N), sig), field)


def test_multi_segment_hub_successors_and_labels():
    # rows longer than one kHeavySegment (1024) segment are reduced
    # segment-wise and combined; successors / centers / labels must equal the
    # oracle's
    n = 9001
    rng = np.random.default_rng(99)
    u, v, _ = H.graphgen.random_edges(n, 3.0, unit=True, seed=99)
    us, vs = [u], [v]
    for h, deg in [(0, 2049), (n - 1, 8000), (4500, 4096), (17, 6000), (n // 3, 2100), (n // 5, 300)]:
        nb = rng.choice(n, size=deg, replace=False)
        nb = nb[nb != h]
        us.append(np.full(len(nb), h, np.int32))
        vs.append(nb.astype(np.int32))
    g = H.G(n, np.concatenate(us), np.concatenate(vs), None, 10.0)
    assert np.diff(g.offsets).max() > 3 * 2048
    sig = [0.3, 1.0, 2.3, 5.0, 12.0, 30.0]
    res, v_dev, succ = N.cluster_sweep(g.csr(N), sig, want_v=True, want_succ=True)
    for q, s in enumerate(sig):
        vo, so, co, cio, ko = O.cluster(g.offsets, g.nbr, g.wt, 10.0, s, workers=4)
        assert_bits(v_dev[q], vo)
        assert np.array_equal(succ[q], so)
        assert np.array_equal(res[q].center, co) and np.array_equal(res[q].cluster_index, cio)
        assert res[q].num_clusters == ko


def test_heavy_row_boundary_degrees():
    """Rows of degree exactly at and one past the GGD heavy-row threshold
    (kHeavyDegree = 256) and at / past one and two heavy segments
    (kHeavySegment = 1024), plus the batched-walk threshold (32): successors,
    centers and labels equal the oracle's (ggd.cpp:7-57)."""
    n = 12001
    rng = np.random.default_rng(7)
    degs = [31, 32, 33, 255, 256, 257, 1023, 1024, 1025, 2047, 2048, 2049, 3072, 3073]
    hubs = np.arange(len(degs), dtype=np.int32) * 7 + 100
    others = np.setdiff1d(np.arange(n, dtype=np.int32), hubs)
    us, vs = [], []
    bu = rng.choice(others, 30000).astype(np.int32)
    bv = rng.choice(others, 30000).astype(np.int32)
    us.append(bu)
    vs.append(bv)
    for h, d in zip(hubs, degs):
        nb = rng.choice(others, size=d, replace=False).astype(np.int32)
        us.append(np.full(d, h, np.int32))
        vs.append(nb)
    g = H.G(n, np.concatenate(us), np.concatenate(vs), None, 10.0)
    assert list(np.diff(g.offsets)[hubs]) == degs
    sig = [0.3, 1.0, 2.3, 5.0, 8.0, 12.0, 20.0, 30.0]
    res, v_dev, succ = N.cluster_sweep(g.csr(N), sig, want_v=True, want_succ=True)
    for q, s in enumerate(sig):
        vo, so, co, cio, ko = O.cluster(g.offsets, g.nbr, g.wt, 10.0, s, workers=8)
        assert_bits(v_dev[q], vo)
        assert np.array_equal(succ[q], so)
        assert np.array_equal(res[q].center, co) and np.array_equal(res[q].cluster_index, cio)
        assert res[q].num_clusters == ko
    # a field that makes every hub its neighbourhood's minimum / maximum
    for vv in (np.arange(n, dtype=np.float64), -np.arange(n, dtype=np.float64)):
        vv = vv.copy()
        vv[hubs] = -1e9 if vv[0] == 0 else 1e9
        assert np.array_equal(N.build_successors(g.csr(N), vv), O.build_successors(g.offsets, g.nbr, vv))


def test_deep_monotone_chain_through_device_ggd():
    """A 1M-node path whose field strictly decreases along it: the successor
    map is ONE chain of depth n - 1 (0 -> 1 -> ... -> n-1, and reversed in the
    second sigma column). The chase stops after its step bound and pointer
    jumping finishes in <= ceil(log2 n) + 2 rounds (ggd.cpp:26-57); before
    the bound, thread 0 alone walked n dependent loads."""
    import time

    import torch
    n = 1 << 20
    g = H.path(n)
    dg = N.DeviceCsr(g.csr(N))
    ar = torch.arange(n, dtype=torch.float64, device="cuda")
    V = torch.stack([float(n) - ar, ar], dim=1).contiguous()  # node-major [n][2]
    succ = torch.empty((2, n), dtype=torch.int32, device="cuda")
    center, ci = torch.empty_like(succ), torch.empty_like(succ)
    nc = torch.empty(2, dtype=torch.int32, device="cuda")
    ws = torch.empty(N.dev_ggd_workspace(n, 2), dtype=torch.uint8, device="cuda")
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        N.dev_ggd(dg, V, 2, succ, center, ci, nc, ws)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
    s = succ.cpu().numpy()
    assert np.array_equal(s[0][:-1], np.arange(1, n)) and s[0][-1] == n - 1
    assert np.array_equal(s[1][1:], np.arange(n - 1)) and s[1][0] == 0
    c = center.cpu().numpy()
    assert np.all(c[0] == n - 1) and np.all(c[1] == 0)
    assert np.all(ci.cpu().numpy() == 0) and list(nc.cpu().numpy()) == [1, 1]
    assert el < 0.5, f"deep chain took {el:.3f} s"


def test_long_path_graph_sweep_properties():
    """gqc_cluster_sweep on a 1M-node path (ties between equal-degree
    interior nodes are broken by rounding noise, so chains of any depth can
    form): GGD outputs satisfy ggd.cpp:7-57's properties over the whole graph."""
    from tests.test_gpu_fullsize import check_ggd
    n = 1 << 20
    g = H.path(n)
    sig = [0.5, 2.0, 5.0, 9.0, 14.0, 20.0, 25.0, 30.0]
    res, v, succ = N.cluster_sweep(g.csr(N), sig, want_v=True, want_succ=True)
    for q in range(len(sig)):
        check_ggd(g.offsets, g.nbr, v[q], succ[q], res[q].center, res[q].cluster_index, res[q].num_clusters)


@pytest.mark.parametrize("kernel,unit,mode", [(N.KERNEL_FASTFWD, False, N.EXP_EIGEN),
                                              (N.KERNEL_FASTFWD, False, N.EXP_GLIBC),
                                              (N.KERNEL_REPLAY, True, N.EXP_EIGEN)])
def test_hub_companion_launch_rows_bitwise(kernel, unit, mode):
    # rows above max(4096, nnz/4096) entries run in the companion launch (own
    # SM) for weighted graphs and the replay kernel; odd n puts the Eigen
    # tail column next to the hub
    setup(kernel, mode)
    n = 8001
    rng = np.random.default_rng(5)
    u, v, w = H.graphgen.random_edges(n, 3.0, unit=unit, seed=5)
    hub = rng.choice(n - 1, size=5000, replace=False) + 1
    hub = np.append(hub[hub != n - 1], n - 1)
    us = np.concatenate([u, np.zeros(len(hub), np.int32)])
    vs = np.concatenate([v, hub.astype(np.int32)])
    ws = None if unit else np.concatenate([w, 0.5 + 1.5 * rng.random(len(hub))])
    g = H.G(n, us, vs, ws, 10.0)
    assert np.diff(g.offsets).max() > 4096
    sig = [0.7, 2.3, 9.0, 30.0] * 2  # 8 sigmas: the warp kernel
    field = N.potentials(g.csr(N), sig)
    for q, s in enumerate(sig[:4]):
        assert_bits(field[q], oracle_field(g, s, mode))


def test_device_binding_follows_stream_and_option():
    # libgqc links its own CUDA runtime: the dev_* entry points bind to the
    # device of the caller's stream (or buffers), host entry points to
    # GQC_OPT_DEVICE; both must agree with torch's view of the device
    import torch
    g = H.random_graph(501, 5.0, seed=4, unit=True)
    dg = N.DeviceCsr(g.csr(N), "cuda:0")
    sig = O.log_sigma_grid(10.0, 8)
    st = torch.cuda.Stream(device="cuda:0")
    out = torch.empty((g.n, len(sig)), dtype=torch.float64, device="cuda:0")
    N.dev_potentials(dg, sig, 0, g.n, out, st)
    st.synchronize()
    N.set_device(0)
    assert N.get_device() == 0
    host = N.potentials(g.csr(N), sig)
    assert_bits(out.cpu().numpy().T.copy(), host)
    out2 = torch.empty_like(out)
    N.dev_potentials(dg, sig, 0, g.n, out2, None)  # legacy default stream: device of the buffers
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int64), out2.view(torch.int64))
    with pytest.raises(ValueError):
        N.set_device(torch.cuda.device_count())


def test_degree_class_order_fast_path_matches_plain_argmin():
    """Opt-in GGD argmin fast path (GQC_CLASS_ORDER=1, launch_class_order):
    on unit-weight graphs the degree classes order the potentials for most
    sigmas and only the best class is gathered. Same successor maps (every
    entry) and labels as the plain argmin (default, a separate process) and
    as the oracle, also on a graph with hub rows (heavy-row argmin next to
    class-ordered light rows) and isolated nodes; the trace shows the verified
    sigmas; weighted fields skip it."""
    import json
    import subprocess
    import sys
    code = r'''
import json, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2305_14641_b200 import native as N
from tests import helpers as H
import hashlib
out = {}
def hub_graph():
    # 20k nodes: 3 hubs of degree ~3000 (above the class cap), 40 of ~150
    # (global-atomic classes), a sparse random rest, 50 isolated nodes
    rng = np.random.default_rng(5)
    n = 20000
    e = set()
    for h, d in [(0, 3100), (7777, 2600), (19999, 3000)] + [(int(x), 150) for x in rng.choice(np.arange(100, 19000), 40, replace=False)]:
        for j in rng.choice(n - 50, d, replace=False):
            if j != h: e.add((min(h, j), max(h, j)))
    for _ in range(60000):
        a, b = rng.integers(0, n - 50, 2)
        if a != b: e.add((min(a, b), max(a, b)))
    rows = [[] for _ in range(n)]
    for a, b in e:
        rows[a].append(b); rows[b].append(a)
    off = np.zeros(n + 1, np.int64); off[1:] = np.cumsum([len(r) for r in rows])
    nbr = np.concatenate([np.sort(np.array(r, np.int32)) for r in rows if r]).astype(np.int32)
    return N.Csr(off, nbr, None, 10.0)
for name, g in [("sbm", None), ("rand", H.random_graph(3001, 14, 21, unit=True)), ("hubs", "hubs"),
                ("weighted", H.random_graph(2001, 9, 22, unit=False))]:
    if g is None:
        off, nbr = H.sbm_csr()
        csr = N.Csr(off, nbr, None, 10.0)
    elif g == "hubs":
        csr = hub_graph()
    else:
        csr = g.csr(N)
    res, _, succ = N.cluster_sweep(csr, np.exp(np.linspace(0.0, np.log(30.0), 32)), want_succ=True)
    out[name] = [hashlib.sha256(succ.tobytes()).hexdigest(), N.last_launch_count(),
                 [r.num_clusters for r in res], hashlib.sha256(b"".join(r.cluster_index.tobytes() for r in res)).hexdigest()]
print(json.dumps(out))
'''
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    runs = {}
    traces = {}
    for flag in ("1", "0"):  # GQC_CLASS_ORDER: on / off
        r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                           env=dict(os.environ, GQC_CLASS_ORDER=flag, GQC_TRACE="1"))
        assert r.returncode == 0, r.stderr[-2000:]
        runs[flag] = json.loads(r.stdout.strip().splitlines()[-1])
        traces[flag] = [ln for ln in r.stderr.splitlines() if "class order:" in ln]
    # three unit-weight sweeps ordered their classes (most sigmas verified)
    assert len(traces["1"]) == 3 and not traces["0"], traces
    for ln in traces["1"]:
        dirs = [int(x) for x in ln.split("dir =")[1].split()]
        assert len(dirs) == 32 and sum(d != 0 for d in dirs) >= 16, ln
    for name in ("sbm", "rand", "hubs", "weighted"):
        on, off = runs["1"][name], runs["0"][name]
        assert on[0] == off[0] and on[2] == off[2] and on[3] == off[3], name
        # the class-order launches ran (unit weights) / were skipped (weighted)
        if name == "weighted":
            assert on[1] == off[1], name
        else:
            assert on[1] > off[1], name
    # and the plain path equals the oracle (sampled sigma)
    g = H.random_graph(3001, 14, 21, unit=True)
    sig = np.exp(np.linspace(0.0, np.log(30.0), 32))
    res, v, succ = N.cluster_sweep(g.csr(N), sig, want_v=True, want_succ=True)
    for q in (0, 9, 31):
        assert np.array_equal(succ[q], O.build_successors(g.offsets, g.nbr, v[q]))


def test_cluster_sweep_intra_counts():
    """gqc_cluster_sweep_intra: modularity's intra-cluster weight per sigma
    (metrics.cpp:37-44) counted on the device, equal to a numpy count over
    the CSR, and the oracle's modularity from those labels; weighted graphs
    are refused."""
    off, nbr = H.sbm_csr()
    csr = N.Csr(off, nbr, None, 10.0)
    sig = O.log_sigma_grid(10.0, 32)
    ci, k, intra = N.cluster_sweep_intra(csr, sig)
    res, _, _ = N.cluster_sweep(csr, sig)
    rows = np.repeat(np.arange(len(off) - 1), np.diff(off))
    for q in (0, 7, 19, 31):
        assert np.array_equal(ci[q], res[q].cluster_index) and k[q] == res[q].num_clusters
        assert intra[q] == int(np.count_nonzero(ci[q][rows] == ci[q][nbr]))
    w = H.random_graph(300, 5, 3, unit=False)
    with pytest.raises(ValueError, match="intra counts need unit weights"):
        N.cluster_sweep_intra(w.csr(N), [1.0])


def test_reserve_then_sweep_same_bits():
    """gqc_reserve sizes the context buffers ahead of a host-API sweep (the
    CLI's warm-up thread): the sweep that follows gives the same bits as one
    without it; bad sizes are GQC_EINVAL."""
    g = H.random_graph(3001, 9, 31, unit=True)
    sig = O.log_sigma_grid(10.0, 16)
    res0, v0, _ = N.cluster_sweep(g.csr(N), sig, want_v=True)
    N.reserve(4000, 2 * 20000, 16)
    res1, v1, _ = N.cluster_sweep(g.csr(N), sig, want_v=True)
    assert np.array_equal(v0.view(np.int64), v1.view(np.int64))
    assert all(np.array_equal(a.cluster_index, b.cluster_index) for a, b in zip(res0, res1))
    for bad in [(0, 10, 1), (10, -1, 1), (10, 10, 0)]:
        with pytest.raises(ValueError):
            N.reserve(*bad)


def test_sparse_graph_takes_16_sigma_argmin_launches_bitwise():
    """A graph whose rows mostly have <= 4 neighbours (R-MAT-like) takes the
    GGD argmin in 16-sigma light-row launches (two rows per warp, chosen from
    a degree sample): every sigma's successor map equals the oracle's, for the
    host-API sweep and for gqc_dev_ggd (the device-CSR sample)."""
    import torch
    g = H.random_graph(6000, 3, 41, unit=True)
    deg = np.diff(g.offsets)
    assert (deg <= 4).mean() > 0.5
    sig = O.log_sigma_grid(10.0, 32)
    res, v, succ = N.cluster_sweep(g.csr(N), sig, want_v=True, want_succ=True)
    for q in range(len(sig)):
        assert np.array_equal(succ[q], O.build_successors(g.offsets, g.nbr, v[q])), q
    dg = N.DeviceCsr(g.csr(N), "cuda:0")
    vn = torch.from_numpy(np.ascontiguousarray(v.T)).to("cuda:0")
    S, n = len(sig), g.n
    s_d = torch.empty((S, n), dtype=torch.int32, device="cuda:0")
    c_d = torch.empty_like(s_d)
    ci_d = torch.empty_like(s_d)
    nc_d = torch.empty(S, dtype=torch.int32, device="cuda:0")
    ws = torch.empty(N.dev_ggd_workspace(n, S), dtype=torch.uint8, device="cuda:0")
    N.dev_ggd(dg, vn, S, s_d, c_d, ci_d, nc_d, ws)
    torch.cuda.synchronize()
    assert np.array_equal(s_d.cpu().numpy(), succ)
    assert all(np.array_equal(ci_d[q].cpu().numpy(), res[q].cluster_index) for q in range(S))
    assert nc_d.cpu().tolist() == [r.num_clusters for r in res]


@pytest.mark.parametrize("n", [6000, 6001])
def test_isolated_rows_instantiation_bitwise(n):
    """Graphs with isolated rows (> 1% of the degree sample) run the
    fast-forward's isolated-row instantiation (numerator a per-sigma
    constant): every potential equals the oracle's bit for bit, including
    isolated rows at columns 0 and n - 1 under the odd-n Eigen tail."""
    rng = np.random.default_rng(n)
    m = n  # avg degree ~2: many isolated rows
    u = rng.integers(1, n - 1, m).astype(np.int32)
    v = rng.integers(1, n - 1, m).astype(np.int32)
    keep = u != v
    g = H.G(n, u[keep], v[keep], None, 10.0)  # rows 0 and n - 1 isolated
    deg = np.diff(g.offsets)
    assert deg[0] == 0 and deg[-1] == 0 and (deg == 0).mean() > 0.05
    sig = O.log_sigma_grid(10.0, 32)
    _, vg, _ = N.cluster_sweep(g.csr(N), sig, want_v=True)
    for q in (0, 5, 11, 20, 31):
        assert_bits(vg[q], O.potentials(g.offsets, g.nbr, g.wt, g.W, sig[q], workers=4))
