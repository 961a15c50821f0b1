"""Python front of bench_tools/graphgen.cpp: seeded benchmark graphs as CSR.

Shapes (BASELINE.json configs):
  sbm_100k()   planted partition, 100 blocks x 1000, avg degree 16, 80% intra
  lfr_1m()     LFR-style, N=1M, avg degree 20 after dedup (stub mean 22.1), tau1=2.5, kmax=1000,
               tau2=1.5, communities [20, 1000], mu=0.3
  rmat_22()    R-MAT scale 22, edge factor 8, (0.57, 0.19, 0.19, 0.05)
All unit weights, W=10, seed 1 by default.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libgraphgen.so")
_lib = None


def build():
    src = os.path.join(HERE, "graphgen.cpp")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(LIB), exist_ok=True)
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-o", LIB, src])
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        P = C.c_void_p
        L.gg_sbm.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_uint64, P, P]
        L.gg_lfr.argtypes = [C.c_int32] + [C.c_double] * 7 + [C.c_uint64, P, P]
        L.gg_rmat.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double, C.c_uint64, P, P]
        L.gg_random_edges.argtypes = [C.c_int32, C.c_double, C.c_int, C.c_uint64, P, P, P, C.c_int64]
        L.gg_random_edges.restype = C.c_int64
        L.gg_copy.argtypes = [P, P]
        L.gg_labels.argtypes = [P]
        _lib = L
    return _lib


def _fetch():
    n = np.zeros(1, np.int32)
    nnz = np.zeros(1, np.int64)
    return n, nnz


def _finish(n, nnz):
    off = np.empty(int(n[0]) + 1, np.int64)
    nbr = np.empty(max(int(nnz[0]), 1), np.int32)
    lib().gg_copy(off.ctypes.data_as(C.c_void_p), nbr.ctypes.data_as(C.c_void_p))
    return off, nbr[: int(nnz[0])]


def sbm(blocks=100, size=1000, avg_deg=16.0, intra=0.8, seed=1):
    n, nnz = _fetch()
    lib().gg_sbm(blocks, size, avg_deg, intra, seed, n.ctypes.data_as(C.c_void_p), nnz.ctypes.data_as(C.c_void_p))
    return _finish(n, nnz)


def lfr(n_nodes=1_000_000, avg_deg=22.1, tau1=2.5, kmax=1000.0, tau2=1.5, cmin=20.0, cmax=1000.0, mu=0.3, seed=1):
    n, nnz = _fetch()
    lib().gg_lfr(n_nodes, avg_deg, tau1, kmax, tau2, cmin, cmax, mu, seed, n.ctypes.data_as(C.c_void_p),
                 nnz.ctypes.data_as(C.c_void_p))
    return _finish(n, nnz)


def rmat(scale=22, edge_factor=8.0, a=0.57, b=0.19, c=0.19, seed=1):
    n, nnz = _fetch()
    lib().gg_rmat(scale, edge_factor, a, b, c, seed, n.ctypes.data_as(C.c_void_p), nnz.ctypes.data_as(C.c_void_p))
    return _finish(n, nnz)


def random_edges(n, avg_deg, unit=False, seed=1):
    """Edge list in the shape of the reference's oracles::random_graph."""
    cap = max(1, int(avg_deg * n / 2.0)) + 1
    u = np.empty(cap, np.int32)
    v = np.empty(cap, np.int32)
    w = np.empty(cap, np.float64)
    m = lib().gg_random_edges(n, avg_deg, 1 if unit else 0, seed, u.ctypes.data_as(C.c_void_p),
                              v.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p), cap)
    return u[:m].copy(), v[:m].copy(), w[:m].copy()


def labels(n):
    """Planted communities of the last sbm()/lfr() graph (int32[n]); call it
    after that generator and before the next one. None for R-MAT."""
    out = np.empty(n, np.int32)
    return out if lib().gg_labels(out.ctypes.data_as(C.c_void_p)) else None


def write_edge_list(path, offsets, nbr):
    """`u v` per undirected edge (u < v) in CSR order."""
    n = len(offsets) - 1
    rows = np.repeat(np.arange(n, dtype=np.int32), np.diff(offsets))
    keep = rows < nbr
    uv = np.stack([rows[keep], nbr[keep]], axis=1)
    with open(path, "w") as f:
        for a in range(0, len(uv), 1 << 20):
            f.write("\n".join(f"{u} {v}" for u, v in uv[a:a + (1 << 20)].tolist()))
            f.write("\n")


sbm_100k = sbm
lfr_1m = lfr
rmat_22 = rmat
