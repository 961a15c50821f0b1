"""ctypes binding of the CPU oracle (oracle/oracle.cpp) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module, and only as the checker or the timed
CPU baseline. The product path (paper_2305_14641_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")

EXP_EIGEN = 0
EXP_GLIBC = 1

_STATUS_EXC = {1: ValueError, 2: IndexError, 3: RuntimeError, 4: OSError, 9: RuntimeError}


class OracleError(Exception):
    pass


def build() -> str:
    """Compile the oracle (g++ -O2 -ffp-contract=off, no -march)."""
    os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
    src = os.path.join(HERE, "oracle.cpp")
    if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", HERE])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


P = C.c_void_p
i32, i64, f64 = C.c_int32, C.c_int64, C.c_double


def _declare(L):
    L.orc_last_error.restype = C.c_char_p
    L.orc_eigen_pexp.restype = f64
    L.orc_eigen_pexp.argtypes = [f64]
    L.orc_glibc_exp.restype = f64
    L.orc_glibc_exp.argtypes = [f64]
    L.orc_csr_from_edges.argtypes = [i32, i64, P, P, P, f64, P, P, P, P]
    L.orc_potentials.argtypes = [i32, P, P, P, f64, f64, C.c_int, C.c_int, P]
    L.orc_potentials_rows.argtypes = [i32, P, P, P, f64, f64, C.c_int, C.c_int, P, i64, P]
    L.orc_potentials_khop.argtypes = [i32, P, P, P, f64, f64, C.c_int, C.c_int, C.c_int, P, i64, P]
    L.orc_build_successors.argtypes = [i32, P, P, P, P]
    L.orc_resolve_centers.argtypes = [i32, P, P, P, P]
    L.orc_log_sigma_grid.argtypes = [f64, C.c_int, f64, f64, P]
    L.orc_linear_sigma_grid.argtypes = [f64, f64, C.c_int, P]
    L.orc_metric_row.argtypes = [i32, P, P, P, f64, P, i32, P, i32, f64, f64, C.c_char_p, i64, P]
    L.orc_run_cluster.argtypes = [C.c_char_p, C.c_char_p, f64, f64, C.c_int, f64, C.c_int,
                                  C.c_char_p, i64, P, C.c_char_p, i64, P]
    L.orc_run_sweep.argtypes = [C.c_char_p, C.c_char_p, f64, C.c_int, f64, f64, f64, C.c_int, C.c_int,
                                C.c_int, C.c_char_p, i64, P, C.c_char_p, i64, P]
    L.orc_detect_mutation.argtypes = [i32, P, P, P, P, P, P]
    L.orc_scores.argtypes = [i64, P, i32, P, i32, P]
    L.orc_modularity.argtypes = [i32, P, P, P, P, f64, P]


def _check(status):
    if status != 0:
        msg = lib().orc_last_error().decode()
        raise _STATUS_EXC.get(status, OracleError)(msg)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def eigen_pexp(x: float) -> float:
    return lib().orc_eigen_pexp(float(x))


def glibc_exp(x: float) -> float:
    return lib().orc_glibc_exp(float(x))


def csr_from_edges(n, u, v, w=None, W=10.0):
    """graph.cpp:25-71 semantics (keep-first dedup, no self loops, ascending rows)."""
    u = np.ascontiguousarray(u, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.int32)
    m = len(u)
    wa = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
    offsets = np.zeros(n + 1, dtype=np.int64)
    nbr = np.zeros(max(2 * m, 1), dtype=np.int32)
    wt = np.zeros(max(2 * m, 1), dtype=np.float64)
    nnz = np.zeros(1, dtype=np.int64)
    _check(lib().orc_csr_from_edges(n, m, _p(u), _p(v), _p(wa), W, _p(offsets), _p(nbr), _p(wt), _p(nnz)))
    k = int(nnz[0])
    return offsets, nbr[:k].copy(), wt[:k].copy()


def potentials(offsets, nbr, wt, W, sigma, workers=1, mode=EXP_EIGEN):
    n = len(offsets) - 1
    out = np.empty(n, dtype=np.float64)
    _check(lib().orc_potentials(n, _p(offsets), _p(nbr), _p(wt), W, sigma, workers, mode, _p(out)))
    return out


def potentials_rows(offsets, nbr, wt, W, sigma, rows, workers=1, mode=EXP_EIGEN):
    n = len(offsets) - 1
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    out = np.empty(len(rows), dtype=np.float64)
    _check(lib().orc_potentials_rows(n, _p(offsets), _p(nbr), _p(wt), W, sigma, workers, mode, _p(rows),
                                     len(rows), _p(out)))
    return out


def potentials_khop(offsets, nbr, wt, W, sigma, hop_cap, workers=1, mode=EXP_EIGEN, rows=None):
    """k-hop distance extension (oracle.cpp fill_khop): d = hops for 2..hop_cap,
    W beyond; hop_cap = 1 is the reference's distance. All rows or a row list."""
    n = len(offsets) - 1
    r = None if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
    out = np.empty(n if r is None else len(r), dtype=np.float64)
    _check(lib().orc_potentials_khop(n, _p(offsets), _p(nbr), _p(wt), W, sigma, hop_cap, workers, mode, _p(r),
                                     0 if r is None else len(r), _p(out)))
    return out


def build_successors(offsets, nbr, v):
    n = len(offsets) - 1
    v = np.ascontiguousarray(v, dtype=np.float64)
    succ = np.empty(n, dtype=np.int32)
    _check(lib().orc_build_successors(n, _p(offsets), _p(nbr), _p(v), _p(succ)))
    return succ


def resolve_centers(succ):
    succ = np.ascontiguousarray(succ, dtype=np.int32)
    n = len(succ)
    center = np.empty(n, dtype=np.int32)
    ci = np.empty(n, dtype=np.int32)
    k = np.zeros(1, dtype=np.int32)
    _check(lib().orc_resolve_centers(n, _p(succ), _p(center), _p(ci), _p(k)))
    return center, ci, int(k[0])


def cluster(offsets, nbr, wt, W, sigma, workers=1, mode=EXP_EIGEN):
    v = potentials(offsets, nbr, wt, W, sigma, workers, mode)
    succ = build_successors(offsets, nbr, v)
    center, ci, k = resolve_centers(succ)
    return v, succ, center, ci, k


def log_sigma_grid(W, steps=30, lo_f=0.1, hi_f=3.0):
    out = np.empty(steps, dtype=np.float64)
    _check(lib().orc_log_sigma_grid(W, steps, lo_f, hi_f, _p(out)))
    return out


def linear_sigma_grid(lo, hi, steps):
    out = np.empty(steps, dtype=np.float64)
    _check(lib().orc_linear_sigma_grid(lo, hi, steps, _p(out)))
    return out


def _strcall(fn, *args, nbuf=1):
    caps = [1 << 16] * nbuf
    while True:
        bufs = [C.create_string_buffer(c) for c in caps]
        lens = [np.zeros(1, dtype=np.int64) for _ in range(nbuf)]
        flat = []
        for b, c, l in zip(bufs, caps, lens):
            flat += [b, c, _p(l)]
        _check(fn(*args, *flat))
        need = [int(l[0]) for l in lens]
        if all(nd < c for nd, c in zip(need, caps)):
            return [b.value.decode() for b in bufs]
        caps = [max(c, nd + 1) for c, nd in zip(caps, need)]


def metric_row(offsets, nbr, wt, W, cluster_index, num_clusters, labels=None, num_classes=0, gamma=1.0,
               sigma=float("nan")):
    n = len(offsets) - 1
    ci = np.ascontiguousarray(cluster_index, dtype=np.int32)
    la = None if labels is None else np.ascontiguousarray(labels, dtype=np.int32)
    (row,) = _strcall(lib().orc_metric_row, n, _p(offsets), _p(nbr), _p(wt), W, _p(ci), num_clusters, _p(la),
                      num_classes, gamma, sigma)
    return row


def run_cluster(graph_path, labels_path, sigma, W=10.0, workers=1, gamma=1.0, mode=EXP_EIGEN):
    a, r = _strcall(lib().orc_run_cluster, graph_path.encode(), (labels_path or "").encode(), sigma, W, workers,
                    gamma, mode, nbuf=2)
    return a, r


def run_sweep(graph_path, labels_path=None, W=10.0, workers=1, gamma=1.0, sigma_min=0.0, sigma_max=0.0,
              steps=30, log_grid=True, mode=EXP_EIGEN):
    s, m = _strcall(lib().orc_run_sweep, graph_path.encode(), (labels_path or "").encode(), W, workers, gamma,
                    sigma_min, sigma_max, steps, 1 if log_grid else 0, mode, nbuf=2)
    return s, m


def detect_mutation(sigmas, counts):
    s = np.ascontiguousarray(sigmas, dtype=np.float64)
    c = np.ascontiguousarray(counts, dtype=np.int32)
    lo, hi = np.zeros(1), np.zeros(1)
    drop, found = np.zeros(1, dtype=np.int32), np.zeros(1, dtype=np.int32)
    _check(lib().orc_detect_mutation(len(s), _p(s), _p(c), _p(lo), _p(hi), _p(drop), _p(found)))
    return (float(lo[0]), float(hi[0]), int(drop[0])) if found[0] else None


def scores(truth, kt, pred, kp):
    t = np.ascontiguousarray(truth, dtype=np.int32)
    p = np.ascontiguousarray(pred, dtype=np.int32)
    out = np.empty(6)
    _check(lib().orc_scores(len(t), _p(t), kt, _p(p), kp, _p(out)))
    return dict(zip(["nmi", "ari", "fmi", "f1", "accuracy", "recall"], out.tolist()))


def modularity(offsets, nbr, wt, clusters, gamma=1.0):
    n = len(offsets) - 1
    c = np.ascontiguousarray(clusters, dtype=np.int32)
    out = np.zeros(1)
    _check(lib().orc_modularity(n, _p(offsets), _p(nbr), _p(wt), _p(c), gamma, _p(out)))
    return float(out[0])
