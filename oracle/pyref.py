"""ctypes binding of the reference's OWN library built in place from
/root/reference/proj/src (oracle/Makefile target `ref` ->
oracle/_ref/libgraphqc_ref.so; Eigen replaced by the restated subset in
oracle/eigen_shim) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may use it, as the checker or the timed CPU baseline. The
prebuilt .so travels to the GPU box; /root/reference does not, so
`available()` is False there when the build was skipped here.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libgraphqc_ref.so")
REF_ROOT = "/root/reference/proj"

_STATUS_EXC = {1: ValueError, 2: IndexError, 3: RuntimeError, 4: OSError, 9: RuntimeError}


class RefError(Exception):
    pass


def build() -> str | None:
    """Compile the reference sources when /root/reference is present."""
    if os.path.isdir(os.path.join(REF_ROOT, "src")):
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"])
    return LIB_PATH if os.path.exists(LIB_PATH) else None


def available() -> bool:
    return os.path.exists(LIB_PATH)


_lib = None
P = C.c_void_p
i32, i64, f64 = C.c_int32, C.c_int64, C.c_double


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_graph_from_csr.restype = P
        L.ref_graph_from_csr.argtypes = [i32, P, P, P, f64]
        L.ref_graph_load.restype = P
        L.ref_graph_load.argtypes = [C.c_char_p, f64]
        L.ref_graph_free.argtypes = [P]
        L.ref_graph_shape.argtypes = [P, P, P]
        L.ref_graph_csr.argtypes = [P, P, P, P]
        L.ref_potentials.argtypes = [P, f64, C.c_int, P]
        L.ref_node_potentials.argtypes = [P, f64, P, i64, C.c_int, P]
        L.ref_ggd.argtypes = [P, f64, P, P, P, P, P]
        L.ref_cluster.argtypes = [P, f64, C.c_int, P, P, P]
        L.ref_resolve.argtypes = [P, i32, P, P, P]
        L.ref_metric_row.argtypes = [P, P, i32, P, i32, f64, f64, C.c_char_p, i64, P]
        L.ref_run_cluster_report.argtypes = [C.c_char_p, C.c_char_p, f64, f64, C.c_int, f64, C.c_char_p, i64, P]
        L.ref_run_sweep.argtypes = [C.c_char_p, C.c_char_p, f64, C.c_int, f64, P, i32, C.c_char_p, i64, P, P, P,
                                    P, P]
        L.ref_log_sigma_grid.argtypes = [f64, C.c_int, f64, f64, P]
        L.ref_array_exp.argtypes = [P, i64, f64, P]
        L.ref_random_graph_seq.restype = P
        L.ref_random_graph_seq.argtypes = [C.c_uint32, P, i32, f64, f64, i32]
        _lib = L
    return _lib


def _check(status):
    if status != 0:
        raise _STATUS_EXC.get(status, RefError)(lib().ref_last_error().decode())


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _strcall(fn, *args):
    cap = 1 << 16
    while True:
        buf = C.create_string_buffer(cap)
        n = np.zeros(1, dtype=np.int64)
        _check(fn(*args, buf, cap, _p(n)))
        if int(n[0]) < cap:
            return buf.value.decode()
        cap = int(n[0]) + 1


class Graph:
    """graphqc::Graph owned by the reference library."""

    def __init__(self, handle):
        self.h = handle
        n, nnz = np.zeros(1, np.int32), np.zeros(1, np.int64)
        _check(lib().ref_graph_shape(self.h, _p(n), _p(nnz)))
        self.n, self.nnz = int(n[0]), int(nnz[0])

    @classmethod
    def from_csr(cls, offsets, nbr, wt, W):
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        nbr = np.ascontiguousarray(nbr, dtype=np.int32)
        wt = None if wt is None else np.ascontiguousarray(wt, dtype=np.float64)
        h = lib().ref_graph_from_csr(len(offsets) - 1, _p(offsets), _p(nbr), _p(wt), W)
        if not h:
            raise ValueError(lib().ref_last_error().decode())
        return cls(h)

    @classmethod
    def random_seq(cls, seed, ns, avg_degree, W=10.0, unit=False):
        """The reference's own oracles::random_graph (tests/oracles.hpp:134-154):
        graphs of ns[0], ns[1], ... nodes drawn in turn from ONE
        std::mt19937(seed); returns the last one."""
        ns = np.ascontiguousarray(ns, dtype=np.int32)
        h = lib().ref_random_graph_seq(seed, _p(ns), len(ns), avg_degree, W, 1 if unit else 0)
        if not h:
            raise ValueError(lib().ref_last_error().decode())
        return cls(h)

    @classmethod
    def load(cls, path, W=10.0):
        h = lib().ref_graph_load(path.encode(), W)
        if not h:
            raise OSError(lib().ref_last_error().decode())
        return cls(h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_graph_free(self.h)
            self.h = None

    def csr(self):
        off = np.zeros(self.n + 1, np.int64)
        nbr = np.zeros(max(self.nnz, 1), np.int32)
        wt = np.zeros(max(self.nnz, 1), np.float64)
        _check(lib().ref_graph_csr(self.h, _p(off), _p(nbr), _p(wt)))
        return off, nbr[: self.nnz], wt[: self.nnz]

    def potentials(self, sigma, workers=1):
        """compute_potentials_parallel (workers=0: compute_potentials)."""
        out = np.empty(self.n, np.float64)
        _check(lib().ref_potentials(self.h, sigma, workers, _p(out)))
        return out

    def node_potentials(self, sigma, rows, threads=1):
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        out = np.empty(len(rows), np.float64)
        _check(lib().ref_node_potentials(self.h, sigma, _p(rows), len(rows), threads, _p(out)))
        return out

    def ggd(self, sigma, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        succ, center, ci = (np.empty(self.n, np.int32) for _ in range(3))
        k = np.zeros(1, np.int32)
        _check(lib().ref_ggd(self.h, sigma, _p(v), _p(succ), _p(center), _p(ci), _p(k)))
        return succ, center, ci, int(k[0])

    def cluster(self, sigma, workers=1):
        center, ci = np.empty(self.n, np.int32), np.empty(self.n, np.int32)
        k = np.zeros(1, np.int32)
        _check(lib().ref_cluster(self.h, sigma, workers, _p(center), _p(ci), _p(k)))
        return center, ci, int(k[0])

    def metric_row(self, cluster_index, num_clusters, labels=None, num_classes=0, gamma=1.0, sigma=float("nan")):
        ci = np.ascontiguousarray(cluster_index, dtype=np.int32)
        la = None if labels is None else np.ascontiguousarray(labels, dtype=np.int32)
        return _strcall(lib().ref_metric_row, self.h, _p(ci), num_clusters, _p(la), num_classes, gamma, sigma)


def resolve(succ):
    succ = np.ascontiguousarray(succ, dtype=np.int32)
    n = len(succ)
    center, ci = np.empty(n, np.int32), np.empty(n, np.int32)
    k = np.zeros(1, np.int32)
    _check(lib().ref_resolve(_p(succ), n, _p(center), _p(ci), _p(k)))
    return center, ci, int(k[0])


def run_cluster_report(graph_path, labels_path, sigma, W=10.0, workers=1, gamma=1.0):
    return _strcall(lib().ref_run_cluster_report, graph_path.encode(), (labels_path or "").encode(), sigma, W,
                    workers, gamma)


def run_sweep(graph_path, sigmas, labels_path=None, W=10.0, workers=1, gamma=1.0):
    """run_sweep + write_sweep_csv; the mutation line in graphqc_main's format."""
    sig = np.ascontiguousarray(sigmas, dtype=np.float64)
    lo, hi = np.zeros(1), np.zeros(1)
    drop, has = np.zeros(1, np.int32), np.zeros(1, np.int32)
    cap = 1 << 20
    buf = C.create_string_buffer(cap)
    n = np.zeros(1, np.int64)
    _check(lib().ref_run_sweep(graph_path.encode(), (labels_path or "").encode(), W, workers, gamma, _p(sig),
                               len(sig), buf, cap, _p(n), _p(lo), _p(hi), _p(drop), _p(has)))
    assert int(n[0]) < cap
    mut = (float(lo[0]), float(hi[0]), int(drop[0])) if has[0] else None
    return buf.value.decode(), mut


def log_sigma_grid(W, steps=30, lo_f=0.1, hi_f=3.0):
    out = np.empty(steps, np.float64)
    _check(lib().ref_log_sigma_grid(W, steps, lo_f, hi_f, _p(out)))
    return out


def array_exp(x, k=1.0):
    """(k * x).exp() of an ArrayXd through the shim (packets + scalar tail)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    _check(lib().ref_array_exp(_p(x), len(x), k, _p(out)))
    return out
