"""The graphqc-compatible CLI (paper_2305_14641_b200/bin/graphqc) against the
reference's CLI contract (tests/cli_test.cpp, README.md) and the oracle.
Commands that never reach the device (eval, parameter/I-O errors, help) run on
CPU; clustering commands are marked gpu and compared byte for byte with the
oracle's restatement of the reference's outputs."""
import math
import os
import subprocess

import numpy as np
import pytest

from oracle import pyoracle as O
from tests import helpers as H

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2305_14641_b200", "bin", "graphqc")
README_ROW = ("0.3122945430637738,0.6486360381182862,0.6684671059738576,0.8319365867687499,"
              "0.9032258064516129,0.9117647058823529,0.8235294117647058,2,5")


def run(*args, stdin=None):
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, input=stdin)
    return r.returncode, r.stdout, r.stderr


def write(path, text):
    path.write_text(text)
    return str(path)


# ------------------------------------------------------------------ CPU only
def test_cli_built():
    assert os.path.exists(CLI), "build with make"


def test_invalid_parameters_exit_2():
    # cli_test.cpp "invalid parameters exit with code 2"
    k = H.KARATE_EDGES
    assert run("cluster", k, "--sigma", "-1")[0] == 2
    assert run("cluster", k, "--sigma", "0")[0] == 2
    assert run("cluster", k, "--sigma", "1", "--workers", "0")[0] == 2
    assert run("cluster", k, "--sigma", "1", "--format", "yaml")[0] == 2
    assert run("nonsense")[0] == 2
    assert run("cluster", k)[0] == 2  # --sigma is required
    assert run("cluster", k, "--sigma", "abc")[0] == 2
    assert run("sweep", k, "--sigma-steps", "0")[0] == 2
    assert run("sweep", k, "--sigma-min", "5", "--sigma-max", "2")[0] == 2
    assert run("bench", "--sizes", "10,5")[0] == 2
    code, out, err = run("cluster", k, "--sigma", "-1")
    assert "sigma must be positive" in err
    for bad in ("0", "8"):  # --hop-cap (k-hop extension, not a reference flag)
        code, out, err = run("cluster", k, "--sigma", "1", "--hop-cap", bad)
        assert code == 2 and "hop-cap must be in 1..7" in err
    assert run("sweep", k, "--hop-cap", "x")[0] == 2


def test_io_failures_exit_1(tmp_path):
    # cli_test.cpp "io failures exit with code 1" (unreadable input)
    assert run("cluster", "/no/such/file.edges", "--sigma", "1")[0] == 1
    bad = write(tmp_path / "bad.edges", "a b\nx\n")
    code, out, err = run("cluster", bad, "--sigma", "1")
    assert code == 1 and "line 2" in err
    assert run("cluster", write(tmp_path / "w.edges", "a b 0\n"), "--sigma", "1")[0] == 1
    assert run("cluster", write(tmp_path / "c.edges", "# only\n\n"), "--sigma", "1")[0] == 1


def test_help_succeeds_and_documents_flags():
    code, out, err = run("cluster", "--help")
    assert code == 0 and "--sigma" in out and "--default-distance" in out
    assert run("--help")[0] == 0


def test_eval_scores_two_labelings(tmp_path):
    # cli_test.cpp "eval scores two labelings"
    t = write(tmp_path / "truth.labels", "a 0\nb 0\nc 1\nd 1\n")
    p = write(tmp_path / "pred.labels", "a 0\nb 0\nc 0\nd 1\n")
    code, out, _ = run("eval", t, t)
    assert code == 0 and ",1,1,1," in out
    code, out, _ = run("eval", t, p)
    row = out.splitlines()[1]
    assert code == 0 and row.startswith(",") and ",0,0.408248290463863" in row
    write(tmp_path / "pred.labels", "a 0\nb 0\nc 0\nq 1\n")
    assert run("eval", t, p)[0] == 2


def test_eval_with_graph_adds_modularity(tmp_path):
    t = write(tmp_path / "t.labels", "0 0\n1 0\n2 1\n3 1\n")
    g = write(tmp_path / "g.edges", "0 1\n1 2\n2 3\n")
    code, out, _ = run("eval", t, t, "--graph", g)
    assert code == 0 and not out.splitlines()[1].startswith(",")


def test_eval_json_format(tmp_path):
    t = write(tmp_path / "t.labels", "a 0\nb 0\nc 1\nd 1\n")
    code, out, _ = run("eval", t, t, "--format", "json")
    assert code == 0
    assert out.strip() == ('{"modularity":null,"nmi":1.0,"ari":1.0,"fmi":1.0,"f1":1.0,"accuracy":1.0,'
                           '"recall":1.0,"num_clusters":2,"sigma":null}')


@pytest.mark.parametrize("seed", [43, 44, 45])
def test_eval_metrics_match_oracle(tmp_path, seed):
    # acceptance criterion 2 shape (seed 43): random labelings, scores vs the oracle, bitwise
    rng = np.random.default_rng(seed)
    for trial in range(20):
        n = int(rng.integers(2, 300))
        kt, kp = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        truth = rng.integers(0, kt, n)
        pred = rng.integers(0, kp, n)
        names = [f"v{i}" for i in range(n)]
        t = write(tmp_path / "t.labels", "".join(f"{a} {b}\n" for a, b in zip(names, truth)))
        p = write(tmp_path / "p.labels", "".join(f"{a} {b}\n" for a, b in zip(names, pred)))
        code, out, _ = run("eval", t, p)
        assert code == 0
        cells = out.splitlines()[1].split(",")
        # dense relabel in first-appearance order (graphqc_main.cpp:284-294)
        def dense(x):
            m = {}
            return np.array([m.setdefault(v, len(m)) for v in x]), len(m)
        td, ktd = dense(truth.tolist())
        pd, kpd = dense(pred.tolist())
        s = O.scores(td, ktd, pd, kpd)
        for col, key in ((1, "nmi"), (2, "ari"), (3, "fmi")):
            assert float(cells[col]) == s[key] or (math.isnan(s[key]) and cells[col] == "")
        if ktd == kpd:
            assert float(cells[4]) == s["f1"] and float(cells[5]) == s["accuracy"] and float(cells[6]) == s["recall"]
        else:
            assert cells[4:7] == ["", "", ""]


def test_eval_modularity_matches_oracle(tmp_path):
    rng = np.random.default_rng(7)
    g = H.random_graph(60, 4.0, seed=3)
    names = [str(i) for i in range(g.n)]
    edges = [(i, int(j), g.wt[k]) for i in range(g.n) for k, j in
             enumerate(g.nbr[g.offsets[i]:g.offsets[i + 1]], start=g.offsets[i]) if i < j]
    gpath = write(tmp_path / "g.edges", "".join(f"{a} {b} {repr(float(w))}\n" for a, b, w in edges))
    labels = rng.integers(0, 3, g.n)
    t = write(tmp_path / "t.labels", "".join(f"{n} {l}\n" for n, l in zip(names, labels)))
    code, out, _ = run("eval", t, t, "--graph", gpath)
    assert code == 0
    # the edge file interns names in first-appearance order; recompute in that order
    order = []
    for a, b, _ in edges:
        for x in (a, b):
            if x not in order:
                order.append(x)
    gg = H.G(len(order), np.array([order.index(a) for a, b, _ in edges]),
             np.array([order.index(b) for a, b, _ in edges]), np.array([w for _, _, w in edges]))
    m = {}
    dense = np.array([m.setdefault(int(labels[x]), len(m)) for x in order])
    q = O.modularity(gg.offsets, gg.nbr, gg.wt, dense)
    assert float(out.splitlines()[1].split(",")[0]) == q


# ---------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_cluster_karate_readme_golden(tmp_path):
    out_csv = tmp_path / "assign.csv"
    code, out, err = run("cluster", H.KARATE_EDGES, "--labels", H.KARATE_LABELS, "--sigma", "5", "--workers", "2",
                         "--out", out_csv)
    assert code == 0, err
    assert out == "modularity,nmi,ari,fmi,f1,accuracy,recall,num_clusters,sigma\n" + README_ROW + "\n"
    a, r = O.run_cluster(H.KARATE_EDGES, H.KARATE_LABELS, 5.0, workers=2)
    assert out_csv.read_text() == a


@pytest.mark.gpu
def test_sweep_karate_mutation_golden(tmp_path):
    out_csv = tmp_path / "sweep.csv"
    code, out, err = run("sweep", H.KARATE_EDGES, "--labels", H.KARATE_LABELS, "--out", out_csv)
    assert code == 0, err
    assert out == "mutation interval: [2.272723014236749, 2.5555343651620004] drop=17\n"
    s, m = O.run_sweep(H.KARATE_EDGES, H.KARATE_LABELS)
    assert out_csv.read_text() == s


@pytest.mark.gpu
def test_sweep_linear_plateau_and_single_point():
    code, out, _ = run("sweep", H.KARATE_EDGES, "--sigma-min", "10", "--sigma-max", "300", "--sigma-steps", "30",
                       "--linear-grid", "--out", "-")
    assert code == 0
    lines = out.strip().splitlines()
    assert lines[-1] == "mutation interval: none"
    assert all(l.split(",")[1] == "2" for l in lines[1:-1]) and len(lines) == 32
    code, out, _ = run("sweep", H.KARATE_EDGES, "--sigma-steps", "1", "--out", "-")
    assert code == 0 and "mutation interval: none" in out


@pytest.mark.gpu
def test_cluster_without_labels_and_json():
    code, out, _ = run("cluster", H.KARATE_EDGES, "--sigma", "5", "--out", "-")
    assert code == 0 and ",,,,,," in out.splitlines()[-1]
    code, out, _ = run("cluster", H.KARATE_EDGES, "--sigma", "5", "--out", "-", "--format", "json")
    assert code == 0 and '"nmi":null' in out and '"recall":null' in out and '"sigma":5.0' in out


@pytest.mark.gpu
def test_outputs_identical_across_workers(tmp_path):
    o1, o2 = tmp_path / "a1.csv", tmp_path / "a2.csv"
    r1 = run("cluster", H.KARATE_EDGES, "--labels", H.KARATE_LABELS, "--sigma", "3", "--out", o1, "--workers", "1")
    r2 = run("cluster", H.KARATE_EDGES, "--labels", H.KARATE_LABELS, "--sigma", "3", "--out", o2, "--workers", "2")
    assert r1[0] == 0 and r2[0] == 0 and r1[1] == r2[1] and o1.read_text() == o2.read_text()
    assert run("cluster", H.KARATE_EDGES, "--sigma", "1", "--out", "/no/such/dir/out.csv")[0] == 1


@pytest.mark.gpu
def test_bench_rows():
    code, out, _ = run("bench", "--sizes", "50,100", "--workers", "1,2", "--out", "-")
    lines = out.strip().splitlines()
    assert code == 0 and lines[0] == "n,workers,serial_ms,parallel_ms,speedup" and len(lines) == 5


@pytest.mark.gpu
def test_weighted_graph_sweep_matches_oracle(tmp_path):
    g = H.random_graph(301, 4.0, seed=5)
    edges = [(i, int(j), g.wt[k]) for i in range(g.n) for k, j in
             enumerate(g.nbr[g.offsets[i]:g.offsets[i + 1]], start=g.offsets[i]) if i < j]
    path = write(tmp_path / "w.edges", "".join(f"{a} {b} {repr(float(w))}\n" for a, b, w in edges))
    out_csv = tmp_path / "s.csv"
    code, out, err = run("sweep", path, "--out", out_csv, "--sigma-steps", "12")
    assert code == 0, err
    s, m = O.run_sweep(path, None, steps=12)
    assert out_csv.read_text() == s and out == m


SMALL_GRAPHS = ["karate_weighted", "les_miserables_weighted", "les_miserables", "florentine", "davis", "planted_4x32"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", SMALL_GRAPHS)
def test_config2_small_graph_sweeps_match_oracle(tmp_path, name):
    # BASELINE config 2 (substitutes): default 30-point log
    # sweep 0.1W..3W on 1 B200, CSV and mutation line byte-identical to the oracle
    path = os.path.join(ROOT, "tests", "golden", f"{name}.edges")
    out_csv = tmp_path / "s.csv"
    code, out, err = run("sweep", path, "--out", out_csv)
    assert code == 0, err
    s, m = O.run_sweep(path, None)
    assert out_csv.read_text() == s and out == m
    for sigma in (1.0, 2.5, 5.0):
        a_csv = tmp_path / "a.csv"
        code, out, err = run("cluster", path, "--sigma", sigma, "--out", a_csv)
        assert code == 0, err
        a, r = O.run_cluster(path, None, sigma)
        assert a_csv.read_text() == a and out == r


@pytest.mark.gpu
def test_cluster_hop_cap_extension(tmp_path):
    """--hop-cap 2 (the opt-in k-hop distance, not a reference feature): the
    assignment equals GGD over the k-hop oracle's field; --hop-cap 1 is the
    README golden again."""
    out_csv = tmp_path / "a.csv"
    code, out, err = run("cluster", H.KARATE_EDGES, "--sigma", "3", "--hop-cap", "2", "--out", out_csv)
    assert code == 0, err
    g, names, _, _ = H.karate()
    v = O.potentials_khop(g.offsets, g.nbr, g.wt, g.W, 3.0, 2, workers=2)
    center, ci, k = O.resolve_centers(O.build_successors(g.offsets, g.nbr, v))
    want = "node,center,cluster\n" + "".join(f"{names[i]},{names[center[i]]},{ci[i]}\n" for i in range(g.n))
    assert out_csv.read_text() == want
    code, out, err = run("cluster", H.KARATE_EDGES, "--labels", H.KARATE_LABELS, "--sigma", "5", "--hop-cap", "1",
                         "--out", tmp_path / "b.csv")
    assert code == 0 and out.splitlines()[1] == README_ROW


@pytest.mark.parametrize("kind", ["int", "mixed", "sparse", "error", "weighted_dups"])
def test_large_edge_files_ingest_like_the_reference(tmp_path, kind):
    """Multi-chunk (> 1 MB) edge files through the parallel loader's paths:
    compact integer names, a non-integer name deep in the file (chunks
    re-parsed in full), sparse huge integer ids (hashed interning) and a bad
    line in a later chunk (first error in file order). Checked through `eval
    --graph` (modularity of a labelling over the loaded graph) against the
    reference's own loader and metrics (oracle/_ref), or the oracle."""
    from oracle import pyref as R
    rng = np.random.default_rng({"int": 1, "mixed": 2, "sparse": 3, "error": 4, "weighted_dups": 5}[kind])
    n, m = (30000, 120000) if kind != "weighted_dups" else (60000, 400000)
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    name = (lambda x: str(x * 70001 + 12345678)) if kind == "sparse" else str
    if kind == "weighted_dups":
        # > 2^18 edges: the host CSR build's multi-threaded counting sorts,
        # with duplicates in both orientations (some with another weight: the
        # first is kept, a warning names it) and self loops (dropped)
        k = m // 20
        src, at = rng.integers(0, m, k), rng.integers(0, m, k)
        flip = rng.random(k) < 0.5
        u[at], v[at] = np.where(flip, v[src], u[src]), np.where(flip, u[src], v[src])
        loops = rng.integers(0, m, m // 100)
        v[loops] = u[loops]
        w = rng.choice([0.5, 1.0, 1.5, 2.0], m)
        lines = [f"{a} {b} {x}\n" for a, b, x in zip(u, v, w)]
    else:
        lines = [f"{name(a)} {name(b)}\n" for a, b in zip(u, v)]
    if kind == "mixed":
        lines[m * 3 // 4] = "node_x 17\n"
    if kind == "error":
        lines[m * 2 // 3] = "1 2 3 4\n"
        lines[m * 5 // 6] = "oops\n"
    gpath = write(tmp_path / "g.edges", "".join(lines))
    assert os.path.getsize(gpath) > (1 << 20)
    if kind == "error":
        code, out, err = run("eval", H.KARATE_LABELS, H.KARATE_LABELS, "--graph", gpath)
        assert code == 1 and f"line {m * 2 // 3 + 1}" in err
        return
    # labels: one class per node in first-appearance order, three classes
    seen = {}
    for ln in lines:
        for t in ln.split()[:2]:
            seen.setdefault(t, len(seen))
    lab = {t: (k * 7) % 3 for t, k in seen.items()}
    lpath = write(tmp_path / "l.labels", "".join(f"{t} {c}\n" for t, c in lab.items()))
    code, out, err = run("eval", lpath, lpath, "--graph", gpath)
    assert code == 0, err
    if kind == "weighted_dups":
        assert "warning: duplicate edge" in err
    if not R.available():
        return
    g = R.Graph.load(gpath)
    ci = np.array([lab[t] for t in seen], dtype=np.int32)
    row = g.metric_row(ci, 3, ci, 3, 1.0)
    assert out.splitlines()[1].split(",")[0] == row.split(",")[0]  # modularity, bit for bit
