"""CPU checks of the drop-in boundary: libgqc.so loads, exports every entry
point include/gqc.h declares, and validates arguments with the reference's
error semantics before touching a device. No compute calls (no GPU here)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gqc.h")
LIB = os.path.join(ROOT, "paper_2305_14641_b200", "libgqc.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gqc_[a-z_]+)\s*\(", text)))


def test_header_declares_the_reference_boundary():
    syms = declared_symbols()
    for s in ["gqc_potentials", "gqc_node_potential", "gqc_build_successors", "gqc_resolve_centers",
              "gqc_cluster_sweep", "gqc_last_error", "gqc_dev_potentials", "gqc_dev_ggd"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build libgqc.so first (make)"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (gqc_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    lib = C.CDLL(LIB)
    for s in declared_symbols():
        assert getattr(lib, s) is not None


def test_library_targets_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_validation_before_device():
    from paper_2305_14641_b200 import native as N
    g = N.Csr(np.array([0, 1, 2], np.int64), np.array([1, 0], np.int32), None, 10.0)
    with pytest.raises(ValueError, match="sigma must be positive"):
        N.potentials(g, [1.0, 0.0])
    with pytest.raises(ValueError, match="sigma must be positive"):
        N.node_potential(g, 0, -1.0)
    with pytest.raises(ValueError, match="workers must be at least 1"):
        N.compute_potentials_parallel(g, 1.0, 0)
    with pytest.raises(ValueError, match="does not match graph size"):
        N.build_successors(g, np.zeros(3))
    with pytest.raises(ValueError, match="unknown exp mode"):
        N.set_exp_mode(7)
    assert N.get_options() == {"exp_mode": 0, "kernel": 0, "hop_cap": 1}
    for bad in (0, 8, -1):
        with pytest.raises(ValueError, match="hop cap must be in 1..7"):
            N.set_hop_cap(bad)
    N.set_hop_cap(3)
    assert N.get_hop_cap() == 3
    N.set_hop_cap(1)
    with pytest.raises(ValueError, match="device ordinal out of range"):
        N.set_device(N.device_count() + 3)
    with pytest.raises(ValueError, match="device ordinal out of range"):
        N.set_device(-1)
    assert N.get_device() == 0


def test_no_cpu_fallback_without_device():
    from paper_2305_14641_b200 import native as N
    if N.device_count() > 0:
        pytest.skip("a GPU is present")
    g = N.Csr(np.array([0, 1, 2], np.int64), np.array([1, 0], np.int32), None, 10.0)
    with pytest.raises(N.CudaError, match="no CUDA device"):
        N.potentials(g, [1.0])


def test_row_shards_partition_cpu():
    """gqc_row_shards (no device needed): contiguous blocks covering every row,
    balanced by deg + 4 per row for the fast-forward kernel, and the
    reference's equal blocks w*floor(n/k) + min(w, n mod k)
    (potential.cpp:70-74) for the dense replay."""
    import numpy as np

    from bench_tools import graphgen
    from paper_2305_14641_b200 import native as N
    graphgen.build()
    off, nbr = graphgen.rmat(scale=16)
    csr = N.Csr(off, nbr, None, 10.0)
    n = len(off) - 1
    cost = np.diff(off) + 4
    for k in (1, 2, 3, 8, 32):
        b = N.row_shards(csr, k)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
        per = np.array([cost[b[r]:b[r + 1]].sum() for r in range(k)])
        assert per.max() <= cost.sum() / k + cost.max()
    N.set_kernel(N.KERNEL_REPLAY)
    try:
        for k in (3, 7):
            b = N.row_shards(csr, k)
            assert list(b) == [w * (n // k) + min(w, n % k) for w in range(k)] + [n]
    finally:
        N.set_kernel(N.KERNEL_FASTFWD)
    import pytest
    with pytest.raises(ValueError):
        N.row_shards(csr, 33)
