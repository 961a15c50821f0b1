"""CPU check of the exact fast-forward algorithm (csrc/ff_chain.cuh, the source
the FASTFWD sm_100a kernel compiles) against naive sequential fp64 adds."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "ff_harness.cpp")
HDR = os.path.join(ROOT, "paper_2305_14641_b200", "csrc", "ff_chain.cuh")
LIB = os.path.join(ROOT, "tests", "_build", "libffharness.so")


@pytest.fixture(scope="module")
def ff():
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(SRC), os.path.getmtime(HDR)):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared",
                               "-I", os.path.dirname(HDR), "-o", LIB, SRC])
    L = C.CDLL(LIB)
    L.fft_single.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_void_p]
    L.fft_single.restype = C.c_longlong
    L.fft_rows.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_void_p]
    L.fft_rows.restype = C.c_longlong
    L.fft_prefix.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_void_p]
    L.fft_prefix.restype = C.c_longlong
    L.fft_rows2.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_void_p]
    L.fft_rows2.restype = C.c_longlong
    L.fft_run.argtypes = [C.c_double, C.c_double, C.c_int]
    L.fft_run.restype = C.c_double
    L.fft_naive.argtypes = [C.c_double, C.c_double, C.c_longlong]
    L.fft_naive.restype = C.c_double
    return L


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_single_runs_bitwise(ff, seed):
    bad = np.zeros(3)
    m = ff.fft_single(seed, 40000, 20000, bad.ctypes.data_as(C.c_void_p))
    assert m == 0, f"{m} mismatches, first (s, c, L) = {bad.tolist()}"


@pytest.mark.parametrize("seed", [11, 12])
def test_row_sequences_bitwise(ff, seed):
    bad = np.zeros(3)
    m = ff.fft_rows(seed, 3000, 20000, bad.ctypes.data_as(C.c_void_p))
    assert m == 0, f"{m} mismatches, first (c, term, row) = {bad.tolist()}"


def test_edge_cases(ff):
    cases = [
        (0.0, 1.0, 1), (0.0, 1.0, 5), (0.0, 0.1, 100000), (1.0, 2.0 ** -53, 1000),  # exact half-ulp tie at 1
        (1.0 + 2.0 ** -52, 2.0 ** -53, 1000),  # odd start, tie: one step to even, then fixed
        (1.0, 3 * 2.0 ** -53, 1000), (2.0 ** 52, 0.5, 10), (2.0 ** 52 + 1, 0.5, 10),
        (0.0, 5e-324, 100000), (0.0, 2.0 ** -1023, 50), (3e-308, 1e-309, 3000),
        (0.0, 0.0, 10), (7.0, 0.0, 10), (1e300, 1e290, 1000), (0.0, 1.9e-22, 999999),
    ]
    for s, c, L in cases:
        a, b = ff.fft_run(s, c, L), ff.fft_naive(s, c, L)
        assert np.float64(a).view(np.int64) == np.float64(b).view(np.int64), (s, c, L, a, b)


@pytest.mark.parametrize("seed", [21, 22])
def test_prefix_segments_bitwise(ff, seed):
    bad = np.zeros(3)
    m = ff.fft_prefix(seed, 300, 30000, bad.ctypes.data_as(C.c_void_p))
    assert m == 0, f"{m} mismatches, first (c, n, L) = {bad.tolist()}"


@pytest.mark.parametrize("seed", [31, 32])
@pytest.mark.parametrize("walk", ["fft_rows2", "fft_rows2w"])
def test_two_chain_rows_with_prefix_bitwise(ff, seed, walk):
    # ff_run2 (pass per chain + general loop) and ff_walk2 (one loop, both chains)
    fn = getattr(ff, walk)
    fn.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_void_p]
    fn.restype = C.c_longlong
    bad = np.zeros(3)
    m = fn(seed, 3000, 20000, bad.ctypes.data_as(C.c_void_p))
    assert m == 0, f"{m} mismatches, first (e, term, row) = {bad.tolist()}"


@pytest.mark.parametrize("seed,ncols", [(21, 200000), (22, 200000), (23, 60), (24, 7), (25, 5000)])
def test_batched_row_walk_bitwise(ff, seed, ncols):
    # walk_events (batched in-binade jumps over neighbour events) vs naive adds
    ff.fft_walk.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    ff.fft_walk.restype = C.c_longlong
    bad = np.zeros(3)
    m = ff.fft_walk(seed, 2000, ncols, bad.ctypes.data_as(C.c_void_p), None)
    assert m == 0, f"{m} mismatches, first (c, c1, row) = {bad.tolist()}"


@pytest.mark.parametrize("seed,ncols,nc", [(31, 5000, 2), (32, 200000, 2), (33, 60, 2), (34, 20000, 3),
                                           (35, 1000000, 2), (36, 7, 3)])
def test_multi_class_batched_walk_bitwise(ff, seed, ncols, nc):
    # walk_events_multi (k-hop extension: one increment per event class) vs naive adds
    ff.fft_walk_multi.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_void_p]
    ff.fft_walk_multi.restype = C.c_longlong
    bad = np.zeros(3)
    m = ff.fft_walk_multi(seed, 1500, ncols, nc, bad.ctypes.data_as(C.c_void_p))
    assert m == 0, f"{m} mismatching rows, first: c={bad[0]!r} c1={bad[1]!r} row={int(bad[2])}"
