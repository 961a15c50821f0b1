"""Test-side graph construction (seeded), mirroring the reference tests'
inputs: oracles::random_graph shapes (tests/oracles.hpp:134-154), stars,
paths, complete graphs, the karate fixture, and small planted partitions.
CSRs are built by the oracle's restatement of graphqc::Graph (graph.cpp:25-71)."""
from __future__ import annotations

import os

import numpy as np

from bench_tools import graphgen
from oracle import pyoracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
KARATE_EDGES = os.path.join(HERE, "golden", "karate.edges")
KARATE_LABELS = os.path.join(HERE, "golden", "karate.labels")


class G:
    """A CSR plus its edge list."""

    def __init__(self, n, u, v, w=None, W=10.0):
        self.n = int(n)
        self.W = float(W)
        self.offsets, self.nbr, wt = O.csr_from_edges(self.n, u, v, w, W)
        self.wt = wt  # always stored (reference stores 1.0 for unit)
        self.unit = w is None or bool(np.all(np.asarray(w) == 1.0))

    def csr(self, native_module, unit_as_null=True):
        w = None if (self.unit and unit_as_null) else self.wt
        return native_module.Csr(self.offsets, self.nbr, w, self.W)


def parse_edge_list(path, W=10.0):
    """graph.cpp:163-190: tokens, '#' comments, names interned in
    first-appearance order, missing weight = 1.0, self loops dropped."""
    names, ids = [], {}
    us, vs, ws = [], [], []

    def intern(t):
        if t not in ids:
            ids[t] = len(names)
            names.append(t)
        return ids[t]

    with open(path) as f:
        for line in f:
            toks = line.split()
            if not toks or toks[0].startswith("#"):
                continue
            w = float(toks[2]) if len(toks) == 3 else 1.0
            a, b = intern(toks[0]), intern(toks[1])
            if a == b:
                continue
            us.append(a)
            vs.append(b)
            ws.append(w)
    return G(len(names), np.array(us), np.array(vs), np.array(ws), W), names


def karate(W=10.0):
    g, names = parse_edge_list(KARATE_EDGES, W)
    labels = {}
    with open(KARATE_LABELS) as f:
        for line in f:
            t = line.split()
            if t and not t[0].startswith("#"):
                labels[t[0]] = t[1]
    classes = {}
    lab = np.array([classes.setdefault(labels[nm], len(classes)) for nm in names], dtype=np.int32)
    return g, names, lab, len(classes)


def random_graph(n, avg_deg, seed, unit=False, W=10.0):
    u, v, w = graphgen.random_edges(n, avg_deg, unit=unit, seed=seed)
    return G(n, u, v, None if unit else w, W)


def star(leaves, W=10.0):
    u = np.zeros(leaves, np.int32)
    v = np.arange(1, leaves + 1, dtype=np.int32)
    return G(leaves + 1, u, v, None, W)


def path(n, W=10.0):
    u = np.arange(n - 1, dtype=np.int32)
    return G(n, u, u + 1, None, W)


def complete(n, W=10.0):
    iu = np.triu_indices(n, 1)
    return G(n, iu[0].astype(np.int32), iu[1].astype(np.int32), None, W)


def planted(groups, size, p_in, p_out, seed, W=10.0):
    rng = np.random.default_rng(seed)
    n = groups * size
    blk = np.arange(n) // size
    iu = np.triu_indices(n, 1)
    same = blk[iu[0]] == blk[iu[1]]
    keep = rng.random(len(iu[0])) < np.where(same, p_in, p_out)
    return G(n, iu[0][keep].astype(np.int32), iu[1][keep].astype(np.int32), None, W)


def sbm_csr(**kw):
    off, nbr = graphgen.sbm(**kw)
    return off, nbr
