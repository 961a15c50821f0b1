"""Warp-level model of the K2 per-event path on LFR rows (dev helper): builds
tools/k2_warp_model.cpp (the same ff_chain.cuh on the host) and reports, per
event of rows with < 32 neighbours and 32 sigma lanes x 2 chains, how often
any lane needs the cache refresh, the crossing branch, a real add, and how
many ff_walk2 trips the warp makes.
    python tools/k2_warp_model.py [rows=3000]"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
from bench_tools import graphgen  # noqa: E402
from oracle import pyoracle as O  # noqa: E402
from paper_2305_14641_b200.sweep import log_sigma_grid  # noqa: E402

so = os.path.join("/tmp", "k2_warp_model.so")
subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-shared", "-fPIC", "-o", so,
                       os.path.join(HERE, "k2_warp_model.cpp")])
lib = C.CDLL(so)
P = C.c_void_p
lib.sim_rows.argtypes = [P, P, P, C.c_int, C.c_int, P, P, P, P, C.c_int, P]
graphgen.build()
off, nbr = graphgen.lfr()
n = len(off) - 1
pW, eW, p1, e1 = [], [], [], []
for s in log_sigma_grid(10.0, 32):
    inv = 1.0 / (2.0 * s * s)
    a, b = O.eigen_pexp(-inv * 100.0), O.eigen_pexp(-inv)
    eW.append(a), pW.append(100.0 * a), e1.append(b), p1.append(b)
pW, eW, p1, e1 = (np.ascontiguousarray(x, np.float64) for x in (pW, eW, p1, e1))
rows = np.random.default_rng(1).choice(n, int(sys.argv[1]) if len(sys.argv) > 1 else 3000, replace=False)
rows = rows.astype(np.int32)
out = np.zeros(9, np.int64)
lib.sim_rows(off.ctypes.data, nbr.ctypes.data, rows.ctypes.data, len(rows), n, pW.ctypes.data, eW.ctypes.data,
             p1.ctypes.data, e1.ctypes.data, 32, out.ctypes.data)
ev, trips, eref, sf, scr, sre, lcr, lre, lref = (int(x) for x in out)
print(f"events {ev}: trips/event {trips / ev:.2f}, events with an entry refresh {eref / ev:.2f}, "
      f"trips with a fast lane {sf / trips:.2f} / a crossing lane {scr / trips:.2f} / a real add {sre / trips:.2f}; "
      f"per event {lcr / ev:.2f} of 64 chains cross, {lref / ev:.2f} refresh, {lre / ev:.2f} real adds")
