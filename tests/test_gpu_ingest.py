"""Device CSR construction (gqc_build_csr) against graph.cpp:25-71 semantics:
the oracle's restatement of graphqc::Graph(n, edges, W) (pinned to the
reference's own loader in test_ref_pin.py), the reference's own loader on a
file through the CLI, and the facade's host build (GQC_HOST_CSR=1 vs
GQC_DEVICE_CSR=1) byte for byte including the duplicate-edge warnings."""
import os
import subprocess

import numpy as np
import pytest

from oracle import pyoracle as O

pytestmark = pytest.mark.gpu

N = pytest.importorskip("paper_2305_14641_b200.native")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2305_14641_b200", "bin", "graphqc")


def edge_list(n, m, seed, weighted, dup_frac=0.05, loop_frac=0.01):
    rng = np.random.default_rng(seed)
    u = rng.integers(0, n, m).astype(np.int32)
    v = rng.integers(0, n, m).astype(np.int32)
    k = int(m * dup_frac)  # re-emit earlier pairs (both orientations), some with another weight
    src = rng.integers(0, m, k)
    flip = rng.random(k) < 0.5
    at = rng.integers(0, m, k)
    u[at] = np.where(flip, v[src], u[src])
    v[at] = np.where(flip, u[src], v[src])
    loops = rng.integers(0, m, int(m * loop_frac))
    v[loops] = u[loops]
    w = None
    if weighted:
        w = rng.choice([0.5, 1.0, 1.5, 2.0], m)
    return u, v, w


@pytest.mark.parametrize("n,m,weighted,seed", [(1, 0, False, 1), (7, 40, True, 2), (1000, 20000, True, 3),
                                               (50000, 400000, False, 4), ((1 << 20) + 3, 3_000_000, True, 5)])
def test_device_csr_matches_oracle(n, m, weighted, seed):
    u, v, w = edge_list(n, m, seed, weighted)
    off, nbr, wt, unit, dups = N.build_csr(n, u, v, w)
    ro, rn, rw = O.csr_from_edges(n, u, v, w, 10.0)
    assert np.array_equal(off, ro) and np.array_equal(nbr, rn)
    assert np.array_equal(wt.view(np.int64), rw.view(np.int64))
    assert unit == bool(np.all(rw == 1.0))
    # conflicting duplicates: every dropped edge whose weight differs from the
    # first occurrence of its pair, ascending input index
    wa = np.ones(m) if w is None else np.asarray(w, np.float64)
    idx = np.flatnonzero(u != v)
    key = np.minimum(u, v).astype(np.int64)[idx] * (n + 1) + np.maximum(u, v)[idx]
    order = np.argsort(key, kind="stable")
    ks, ids = key[order], idx[order]
    head = np.ones(len(ks), bool)
    head[1:] = ks[1:] != ks[:-1]
    first_of = ids[np.maximum.accumulate(np.where(head, np.arange(len(ks)), 0))] if len(ks) else ids
    conf = ~head & (wa[ids] != wa[first_of])
    want = sorted(zip(ids[conf].tolist(), first_of[conf].tolist()))
    assert dups == want[: len(dups)] and len(dups) == min(len(want), 1 << 16)


def test_device_csr_errors_in_input_order():
    u = np.array([0, 1, 5, 2], np.int32)
    v = np.array([1, 2, 1, 9], np.int32)
    with pytest.raises(IndexError, match="edge endpoint out of range"):
        N.build_csr(6, u, v, np.array([1.0, 1.0, 1.0, 1.0]))
    with pytest.raises(ValueError, match="edge weight must be positive"):
        N.build_csr(10, u, v, np.array([1.0, -1.0, 1.0, 1.0]))
    # an out-of-range endpoint before a bad weight, and vice versa
    with pytest.raises(IndexError):
        N.build_csr(6, u, v, np.array([1.0, 1.0, 1.0, 0.0]))
    with pytest.raises(ValueError):
        N.build_csr(6, u, v, np.array([1.0, 0.0, 1.0, 1.0]))


def run_cli(args, env_extra):
    env = dict(os.environ, **env_extra)
    p = subprocess.run([CLI] + [str(a) for a in args], capture_output=True, text=True, env=env)
    return p.returncode, p.stdout, p.stderr


def test_cli_device_build_equals_host_build_and_reference(tmp_path):
    """A 1.2M-line edge file (string and integer names, duplicates with other
    weights, self loops): `graphqc cluster` gives the same report, assignment
    and duplicate warnings with the device CSR build and the host build, and
    `eval --graph` gives the reference loader's modularity bit for bit."""
    from oracle import pyref as R
    n, m = 200_000, 1_200_000
    u, v, w = edge_list(n, m, 12, True)
    names = np.array([f"n{i}" if i % 7 == 0 else str(i) for i in range(n)])
    lines = [f"{names[a]} {names[b]} {x}\n" for a, b, x in zip(u, v, w)]
    gpath = tmp_path / "g.edges"
    with open(gpath, "w") as f:
        f.write("".join(lines))
    outs = []
    for host in ("1", "0"):
        out_csv = tmp_path / f"a{host}.csv"
        code, out, err = run_cli(["cluster", gpath, "--sigma", "3", "--out", out_csv],
                                 {"GQC_HOST_CSR": host, "GQC_DEVICE_CSR": "0" if host == "1" else "1"})
        assert code == 0, err
        outs.append((out, err, open(out_csv).read()))
    assert outs[0] == outs[1]
    assert "warning: duplicate edge" in outs[0][1]
    # modularity of a labelling over the loaded graph vs the reference's loader
    seen = {}
    for ln in lines:
        for t in ln.split()[:2]:
            seen.setdefault(t, len(seen))
    lab = {t: (k * 7) % 3 for t, k in seen.items()}
    lpath = tmp_path / "l.labels"
    with open(lpath, "w") as f:
        f.write("".join(f"{t} {c}\n" for t, c in lab.items()))
    code, out, err = run_cli(["eval", lpath, lpath, "--graph", gpath], {"GQC_DEVICE_CSR": "1"})
    assert code == 0, err
    if R.available():
        g = R.Graph.load(str(gpath))
        ci = np.array([lab[t] for t in seen], dtype=np.int32)
        row = g.metric_row(ci, 3, ci, 3, 1.0)
        assert out.splitlines()[1].split(",")[0] == row.split(",")[0]
