"""Reference acceptance criterion 5 (joint scale invariance) and default
distances W != 10, on the reference's own code and on the sm_100a path.

Criterion 5 (/root/reference/proj/tests/acceptance_test.cpp:202-248,
potential_test.cpp:105-118): 8 random-weight graphs of 40 + 25 * trial nodes
drawn from ONE std::mt19937(46) by the reference's own generator
(oracles::random_graph, tests/oracles.hpp:134-154, compiled into oracle/_ref);
sigma = 2.3; for c in {0.5, 3, 100} the weights, W and sigma are scaled by c.
The fields must agree to 1e-12 relative, and the successor maps and the
assignments must be identical. Karate (unit weights) gets the value check.

Scaling W moves every per-sigma constant of the path: e_W = exp(-W^2/2s^2),
p_W = W^2 e_W (potential.cpp:19-35) — at W = 1000 with sigma in the default
grid e_W is 0 or subnormal — and W < 1 puts the non-adjacent distance BELOW
the edge weights. Every case is compared bit for bit with the reference's
own build (oracle/_ref), through both the batched (>= 8 sigmas, warp per row)
and the single-sigma (thread per row) kernels and through both potential
kernels (fast-forward, dense replay).

CPU tests pin the oracle restatement on the same inputs; GPU tests
(@pytest.mark.gpu) call the C-ABI."""
import numpy as np
import pytest

from oracle import pyoracle as O
from oracle import pyref as R
from tests import helpers as H

needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")

SCALES = (0.5, 3.0, 100.0)
SIGMA = 2.3
TRIALS = 8


def rel_diff(a, b):
    """acceptance_test.cpp's rel_diff: |a - b| / max(|a|, |b|, tiny)."""
    return np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-300)


def criterion5_graph(trial):
    """(off, nbr, w) of the reference's trial-th criterion-5 graph."""
    g = R.Graph.random_seq(46, [40 + 25 * t for t in range(trial + 1)], 4.0, W=10.0)
    return g.csr()


def scaled_ref(off, nbr, w, W, c):
    """graphqc::Graph(n, scaled edges, c * W) (acceptance_test.cpp:219-221)."""
    return R.Graph.from_csr(off, nbr, w * c, c * W)


def assert_bits(a, b, what=""):
    a, b = np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64)
    bad = np.flatnonzero(a.view(np.int64) != b.view(np.int64))
    assert bad.size == 0, f"{what}: {bad.size} mismatches at {bad[:5]}"


# ------------------------------------------------------------------ CPU ----

@needs_ref
@pytest.mark.parametrize("trial", range(TRIALS))
def test_criterion5_reference_and_oracle_agree(trial):
    """The reference's own code passes criterion 5 here, and the oracle
    restatement reproduces its fields and maps bit for bit at every scale."""
    off, nbr, w = criterion5_graph(trial)
    rg = R.Graph.from_csr(off, nbr, w, 10.0)
    v0 = rg.potentials(SIGMA, 1)
    assert_bits(O.potentials(off, nbr, w, 10.0, SIGMA), v0, "oracle vs reference, c=1")
    s0, c0, ci0, _ = rg.ggd(SIGMA, v0)
    for c in SCALES:
        h = scaled_ref(off, nbr, w, 10.0, c)
        v1 = h.potentials(c * SIGMA, 1)
        assert np.all(rel_diff(v0, v1) <= 1e-12)
        assert_bits(O.potentials(off, nbr, w * c, 10.0 * c, c * SIGMA), v1, f"oracle vs reference, c={c}")
        s1, c1, ci1, _ = h.ggd(c * SIGMA, v1)
        assert np.array_equal(s1, s0) and np.array_equal(c1, c0) and np.array_equal(ci1, ci0)


W_CASES = (0.5, 3.0, 1000.0)


def unit_and_weighted_graphs():
    """Unit graphs (odd and even N: the Eigen tail column) and a weighted one
    whose weights straddle W = 0.5."""
    return [H.random_graph(301, 6, 21, unit=True), H.random_graph(512, 9, 22, unit=True),
            H.random_graph(257, 5, 23, unit=False)]


@needs_ref
@pytest.mark.parametrize("W", W_CASES)
def test_default_distance_oracle_pinned(W):
    for g in unit_and_weighted_graphs():
        wt = None if g.unit else g.wt
        rg = R.Graph.from_csr(g.offsets, g.nbr, wt, W)
        for s in np.concatenate([R.log_sigma_grid(W, 6), [0.05, 1.0, 300.0]]):
            assert_bits(O.potentials(g.offsets, g.nbr, wt, W, s), rg.potentials(s, 1), f"W={W} sigma={s}")


# ------------------------------------------------------------------ GPU ----

def _gpu():
    return pytest.importorskip("paper_2305_14641_b200.native")


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("kernel", ["fastfwd", "replay"])
def test_criterion5_gpu(kernel):
    """Criterion 5 on the GPU: each scaled field equals the reference's own
    field bit for bit (hence the 1e-12 invariance), and the successor maps
    and assignments are invariant, through gqc_cluster_sweep."""
    N = _gpu()
    N.set_kernel(N.KERNEL_REPLAY if kernel == "replay" else N.KERNEL_FASTFWD)
    try:
        for trial in range(TRIALS):
            off, nbr, w = criterion5_graph(trial)
            base = None
            for c in (1.0,) + SCALES:
                rg = R.Graph.from_csr(off, nbr, w * c, 10.0 * c)
                v_ref = rg.potentials(c * SIGMA, 1)
                s_ref, c_ref, ci_ref, k_ref = rg.ggd(c * SIGMA, v_ref)
                # one sigma (thread-per-row kernel) and a batch of 8 around it (warp kernel)
                one = N.cluster(N.Csr(off, nbr, w * c, 10.0 * c), c * SIGMA)
                sig = c * np.array([0.4, 0.9, 1.7, SIGMA, 3.1, 7.0, 12.0, 40.0])
                res, v, succ = N.cluster_sweep(N.Csr(off, nbr, w * c, 10.0 * c), sig, want_v=True, want_succ=True)
                assert_bits(v[3], v_ref, f"trial {trial} c={c}")
                assert np.array_equal(succ[3], s_ref)
                for r in (one, res[3]):
                    assert np.array_equal(r.center, c_ref) and np.array_equal(r.cluster_index, ci_ref)
                    assert r.num_clusters == k_ref
                if base is None:
                    base = (v_ref, s_ref, c_ref, ci_ref)
                else:
                    assert np.all(rel_diff(base[0], v[3]) <= 1e-12)
                    assert np.array_equal(succ[3], base[1])
                    assert np.array_equal(res[3].center, base[2]) and np.array_equal(res[3].cluster_index, base[3])
    finally:
        N.set_kernel(N.KERNEL_FASTFWD)


@pytest.mark.gpu
@needs_ref
def test_criterion5_karate_values_gpu():
    N = _gpu()
    g, _, _, _ = H.karate()
    base = None
    for c in (1.0,) + SCALES:
        rg = R.Graph.from_csr(g.offsets, g.nbr, g.wt * c, 10.0 * c)
        v_ref = rg.potentials(2.3 * c, 1)
        v = N.potentials(N.Csr(g.offsets, g.nbr, g.wt * c, 10.0 * c), [2.3 * c])[0]
        assert_bits(v, v_ref, f"karate c={c}")
        if base is None:
            base = v
        assert np.all(rel_diff(base, v) <= 1e-12)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("W", W_CASES)
@pytest.mark.parametrize("kernel", ["fastfwd", "replay"])
def test_default_distance_gpu_bitwise(W, kernel):
    """W in {0.5, 3, 1000} (pW = W^2 e_W subnormal or 0 at W = 1000; W below
    the edge weights at 0.5): fields, successor maps and labels equal the
    reference's own, for the default log grid 0.1W..3W plus fixed sigmas."""
    N = _gpu()
    N.set_kernel(N.KERNEL_REPLAY if kernel == "replay" else N.KERNEL_FASTFWD)
    try:
        for g in unit_and_weighted_graphs():
            wt = None if g.unit else g.wt
            rg = R.Graph.from_csr(g.offsets, g.nbr, wt, W)
            sig = np.concatenate([[0.05, 1.0], R.log_sigma_grid(W, 30), [300.0, 5000.0]])
            sig = np.unique(sig)
            res, v, succ = N.cluster_sweep(N.Csr(g.offsets, g.nbr, wt, W), sig, want_v=True, want_succ=True)
            for q, s in enumerate(sig):
                v_ref = rg.potentials(s, 1)
                assert_bits(v[q], v_ref, f"W={W} sigma={s}")
                s_ref, c_ref, ci_ref, k_ref = rg.ggd(s, v_ref)
                assert np.array_equal(succ[q], s_ref), f"W={W} sigma={s}"
                assert np.array_equal(res[q].cluster_index, ci_ref) and res[q].num_clusters == k_ref
            for s in (sig[0], sig[len(sig) // 2], sig[-1]):  # single-sigma kernel
                one = N.cluster(N.Csr(g.offsets, g.nbr, wt, W), s)
                _, c_ref, ci_ref, k_ref = rg.ggd(s, rg.potentials(s, 1))
                assert np.array_equal(one.cluster_index, ci_ref) and one.num_clusters == k_ref
    finally:
        N.set_kernel(N.KERNEL_FASTFWD)
