"""ctypes binding of libgqc (include/gqc.h), the B200 hot path.

Mirrors the reference's potential / GGD interface (proj/include/graphqc/
potential.hpp:29-37, ggd.hpp:28-37) on numpy arrays:

    compute_potentials(g, sigma)              -> np.ndarray[N]        (potential.hpp:33)
    compute_potentials_parallel(g, sigma, w)  -> np.ndarray[N]        (potential.hpp:37)
    potentials(g, sigmas)                     -> np.ndarray[S, N]     (batched over sigma)
    node_potential(g, node, sigma)            -> float                (potential.hpp:30)
    build_successors(g, v)                    -> np.ndarray[N] int32  (ggd.hpp:28)
    resolve_centers(succ)                     -> ClusterAssignment    (ggd.hpp:33)
    cluster(g, sigma, workers=1)              -> ClusterAssignment    (ggd.hpp:37)
    cluster_sweep(g, sigmas)                  -> list[ClusterAssignment]

Errors follow the reference's exception classes: std::invalid_argument ->
ValueError, std::out_of_range -> IndexError, std::logic_error -> LogicError
(a RuntimeError), with the reference's messages. There is no CPU fallback:
if libgqc.so is missing the import fails, and without a GPU every compute call
raises CudaError.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgqc.so")

EXP_EIGEN = 0
EXP_GLIBC = 1
KERNEL_FASTFWD = 0
KERNEL_REPLAY = 1
_OPT_EXP_MODE = 1
_OPT_KERNEL = 2
_OPT_GPUS = 5
_OPT_DEVICE = 3
_OPT_HOP_CAP = 4


class GqcError(Exception):
    status = -1


class LogicError(RuntimeError):
    """std::logic_error (e.g. 'successor map contains a cycle')."""


class CudaError(RuntimeError):
    pass


class IoError(OSError):
    pass


_STATUS = {1: ValueError, 2: IndexError, 3: LogicError, 4: IoError, 5: CudaError, 6: MemoryError, 7: CudaError}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
            "the hot path has no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    P, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    lib.gqc_last_error.restype = C.c_char_p
    lib.gqc_version.restype = C.c_char_p
    lib.gqc_last_launch_count.restype = i64
    lib.gqc_device_count.restype = i32
    for name, args in {
        "gqc_set_option": [C.c_int, i64],
        "gqc_get_option": [C.c_int, P],
        "gqc_potentials": [P, P, i32, P],
        "gqc_node_potential": [P, i32, f64, P],
        "gqc_build_successors": [P, P, P],
        "gqc_resolve_centers": [i32, P, P, P, P],
        "gqc_cluster_sweep": [P, P, i32, P, P, P, P, P],
        "gqc_cluster_sweep_intra": [P, P, i32, P, P, P, P, P, P],
        "gqc_cluster_sweep_multi": [P, P, i32, P, i32, P, P, P, P, P, P],
        "gqc_potentials_multi": [P, P, i32, P, i32, P],
        "gqc_row_shards": [P, i32, P],
        "gqc_build_csr": [i32, i64, P, P, P, P, P, P, P, i64, P],
        "gqc_dev_potentials_peer": [P, P, i32, i32, i32, P, i32, i32, P],
        "gqc_ipc_alloc": [C.c_size_t, P, P],
        "gqc_ipc_open": [P, P],
        "gqc_ipc_close": [P],
        "gqc_ipc_free": [P],
        "gqc_dev_potentials": [P, P, i32, i32, i32, P, P],
        "gqc_dev_potentials_packed": [P, P, i32, i32, i32, P, i32, i64, P],
        "gqc_dev_ggd": [P, P, i32, P, P, P, P, P, C.c_size_t, P],
        "gqc_dev_transpose": [P, i32, i32, P, P],
        "gqc_dev_successors": [P, P, i32, i32, i32, P, P],
        "gqc_dev_resolve": [i32, i32, P, P, P, P, P, C.c_size_t, P],
        "gqc_reserve": [i32, i64, i32],
    }.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.gqc_dev_ggd_workspace.argtypes = [i32, i32]
    lib.gqc_dev_ggd_workspace.restype = C.c_size_t
    lib.gqc_dev_resolve_workspace.argtypes = [i32, i32]
    lib.gqc_dev_resolve_workspace.restype = C.c_size_t
    return lib


_lib = _load()


def lib():
    return _lib


def _check(status: int):
    if status != 0:
        msg = _lib.gqc_last_error().decode()
        raise _STATUS.get(status, GqcError)(msg)


class _GqcCsr(C.Structure):
    _fields_ = [("n", C.c_int32), ("nnz", C.c_int64), ("offsets", C.c_void_p), ("nbr", C.c_void_p),
                ("w", C.c_void_p), ("W", C.c_double)]


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class Csr:
    """graphqc::Graph's CSR (graph.hpp:66-71): int64 offsets, int32 ascending
    neighbour ids, float64 weights (None = unit), default distance W."""
    offsets: np.ndarray
    nbr: np.ndarray
    w: Optional[np.ndarray] = None
    W: float = 10.0

    def __post_init__(self):
        self.offsets = np.ascontiguousarray(self.offsets, dtype=np.int64)
        self.nbr = np.ascontiguousarray(self.nbr, dtype=np.int32)
        if self.w is not None:
            self.w = np.ascontiguousarray(self.w, dtype=np.float64)

    @property
    def n(self) -> int:
        return len(self.offsets) - 1

    @property
    def nnz(self) -> int:
        return len(self.nbr)

    def c_struct(self) -> _GqcCsr:
        return _GqcCsr(self.n, self.nnz, _ptr(self.offsets).value, _ptr(self.nbr).value if self.nnz else None,
                       None if self.w is None else _ptr(self.w).value, float(self.W))

    def check_node(self, i: int):
        if i < 0 or i >= self.n:
            raise IndexError(f"node id {i} out of range")


@dataclass
class ClusterAssignment:
    """graphqc::ClusterAssignment (ggd.hpp:21-26)."""
    center: np.ndarray
    cluster_index: np.ndarray
    num_clusters: int
    centers: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.centers is None:
            idx = np.arange(len(self.center), dtype=np.int32)
            self.centers = idx[self.center == idx]


def set_exp_mode(mode: int):
    _check(_lib.gqc_set_option(_OPT_EXP_MODE, int(mode)))


def set_kernel(kernel: int):
    _check(_lib.gqc_set_option(_OPT_KERNEL, int(kernel)))


def set_device(device: int):
    """CUDA device of the host-buffer entry points (potentials, cluster_sweep,
    ...). The dev_* functions follow the device of the stream they are given.
    libgqc has its own CUDA runtime: torch.cuda.set_device does not reach it."""
    _check(_lib.gqc_set_option(_OPT_DEVICE, int(device)))


def set_gpus(g: int):
    """GQC_OPT_GPUS: the host-buffer sweeps (potentials, cluster_sweep, ...)
    run row-sharded on devices GQC_OPT_DEVICE .. + g - 1; same bits for any g."""
    _check(_lib.gqc_set_option(_OPT_GPUS, int(g)))


def get_gpus() -> int:
    v = np.zeros(1, dtype=np.int64)
    _check(_lib.gqc_get_option(_OPT_GPUS, _ptr(v)))
    return int(v[0])


def set_hop_cap(k: int):
    """Distance model of the potential entry points: 1 = the reference's
    (graph.cpp:258-267); 2..7 = the opt-in k-hop extension (BFS hop counts up
    to k, W beyond; unit-weight graphs only). Not a reference feature."""
    _check(_lib.gqc_set_option(_OPT_HOP_CAP, int(k)))


def get_hop_cap() -> int:
    v = np.zeros(1, dtype=np.int64)
    _check(_lib.gqc_get_option(_OPT_HOP_CAP, _ptr(v)))
    return int(v[0])


def get_device() -> int:
    v = np.zeros(1, dtype=np.int64)
    _check(_lib.gqc_get_option(_OPT_DEVICE, _ptr(v)))
    return int(v[0])


def get_options():
    v = np.zeros(1, dtype=np.int64)
    _check(_lib.gqc_get_option(_OPT_EXP_MODE, _ptr(v)))
    mode = int(v[0])
    _check(_lib.gqc_get_option(_OPT_KERNEL, _ptr(v)))
    kernel = int(v[0])
    _check(_lib.gqc_get_option(_OPT_HOP_CAP, _ptr(v)))
    return {"exp_mode": mode, "kernel": kernel, "hop_cap": int(v[0])}


def device_count() -> int:
    return int(_lib.gqc_device_count())


def reserve(n: int, nnz: int, n_sigma: int):
    """gqc_reserve: size the device context's buffers for host-API sweeps of
    graphs up to n nodes / nnz entries / n_sigma sigmas per call."""
    _check(_lib.gqc_reserve(int(n), int(nnz), int(n_sigma)))


def last_launch_count() -> int:
    return int(_lib.gqc_last_launch_count())


def potentials(g: Csr, sigmas: Sequence[float]) -> np.ndarray:
    s = np.ascontiguousarray(np.atleast_1d(np.asarray(sigmas, dtype=np.float64)))
    out = np.empty((len(s), g.n), dtype=np.float64)
    cs = g.c_struct()
    _check(_lib.gqc_potentials(C.byref(cs), _ptr(s), len(s), _ptr(out)))
    return out


def compute_potentials(g: Csr, sigma: float) -> np.ndarray:
    return potentials(g, [sigma])[0]


def compute_potentials_parallel(g: Csr, sigma: float, workers: int) -> np.ndarray:
    """The reference's thread count has no device meaning; it is validated
    exactly as potential.cpp:64 does and the field is the same bits."""
    if not (sigma > 0.0):
        raise ValueError("sigma must be positive")
    if workers < 1:
        raise ValueError("workers must be at least 1")
    return compute_potentials(g, sigma)


def node_potential(g: Csr, node: int, sigma: float) -> float:
    out = np.zeros(1)
    cs = g.c_struct()
    _check(_lib.gqc_node_potential(C.byref(cs), int(node), float(sigma), _ptr(out)))
    return float(out[0])


def build_successors(g: Csr, v: np.ndarray) -> np.ndarray:
    v = np.ascontiguousarray(v, dtype=np.float64)
    if v.shape != (g.n,):
        raise ValueError("potential field does not match graph size")  # ggd.cpp:9-10
    succ = np.empty(g.n, dtype=np.int32)
    cs = g.c_struct()
    _check(_lib.gqc_build_successors(C.byref(cs), _ptr(v), _ptr(succ)))
    return succ


def resolve_centers(succ: np.ndarray) -> ClusterAssignment:
    succ = np.ascontiguousarray(succ, dtype=np.int32)
    n = len(succ)
    center = np.empty(n, dtype=np.int32)
    ci = np.empty(n, dtype=np.int32)
    k = np.zeros(1, dtype=np.int32)
    _check(_lib.gqc_resolve_centers(n, _ptr(succ), _ptr(center), _ptr(ci), _ptr(k)))
    return ClusterAssignment(center, ci, int(k[0]))


def cluster_sweep_raw(g: Csr, sigmas: np.ndarray, center: Optional[np.ndarray], ci: np.ndarray, k: np.ndarray,
                      v: Optional[np.ndarray] = None, succ: Optional[np.ndarray] = None):
    """gqc_cluster_sweep into caller-owned (e.g. pinned) sigma-major arrays."""
    cs = g.c_struct()
    _check(_lib.gqc_cluster_sweep(C.byref(cs), _ptr(sigmas), len(sigmas), _ptr(v), _ptr(succ), _ptr(center),
                                  _ptr(ci), _ptr(k)))


def cluster_sweep_intra(g: Csr, sigmas: Sequence[float]):
    """Labels, counts and modularity's intra-cluster weight per sigma
    (gqc_cluster_sweep_intra; unit-weight graphs)."""
    s = np.ascontiguousarray(np.atleast_1d(np.asarray(sigmas, dtype=np.float64)))
    ci = np.empty((len(s), g.n), dtype=np.int32)
    k = np.zeros(len(s), dtype=np.int32)
    intra = np.zeros(len(s), dtype=np.int64)
    cs = g.c_struct()
    _check(_lib.gqc_cluster_sweep_intra(C.byref(cs), _ptr(s), len(s), None, None, None, _ptr(ci), _ptr(k),
                                        _ptr(intra)))
    return ci, k, intra


def cluster_sweep(g: Csr, sigmas: Sequence[float], want_v: bool = False, want_succ: bool = False,
                  want_center: bool = True):
    """One ClusterAssignment per sigma (the per-sigma body of run_sweep,
    sweep.cpp:50-57); optionally the potential fields and successor maps.
    want_center=False skips the center arrays (centers still listed)."""
    s = np.ascontiguousarray(np.atleast_1d(np.asarray(sigmas, dtype=np.float64)))
    S, n = len(s), g.n
    v = np.empty((S, n)) if want_v else None
    succ = np.empty((S, n), dtype=np.int32) if want_succ else None
    center = np.empty((S, n), dtype=np.int32) if want_center else None
    ci = np.empty((S, n), dtype=np.int32)
    k = np.zeros(S, dtype=np.int32)
    cluster_sweep_raw(g, s, center, ci, k, v, succ)
    if center is None:
        out = [ClusterAssignment(None, ci[q], int(k[q]), centers=np.zeros(0, np.int32)) for q in range(S)]
    else:
        out = [ClusterAssignment(center[q], ci[q], int(k[q])) for q in range(S)]
    return out, v, succ


def build_csr(n: int, u, v, w=None, dup_cap: int = 1 << 16):
    """gqc_build_csr: graphqc::Graph's CSR (graph.cpp:25-71) from an edge list
    in input order, on the device. Returns (offsets, nbr, weights, unit,
    dups) with dups = [(dropped, kept)] input indices of conflicting duplicates."""
    m = len(u)
    e = np.zeros(m, dtype=[("u", np.int32), ("v", np.int32), ("w", np.float64)])
    e["u"], e["v"] = u, v
    e["w"] = 1.0 if w is None else w
    off = np.zeros(n + 1, dtype=np.int64)
    nbr = np.zeros(max(1, 2 * m), dtype=np.int32)
    wt = np.zeros(max(1, 2 * m), dtype=np.float64)
    nnz, unit, nd = np.zeros(1, np.int64), np.zeros(1, np.int32), np.zeros(1, np.int64)
    dup = np.zeros(2 * dup_cap, dtype=np.int64)
    _check(_lib.gqc_build_csr(int(n), m, _ptr(e), _ptr(off), _ptr(nbr), _ptr(wt), _ptr(nnz), _ptr(unit), _ptr(dup),
                              dup_cap, _ptr(nd)))
    k = int(nnz[0])
    d = int(min(nd[0], dup_cap))
    return off, nbr[:k], wt[:k], bool(unit[0]), [(int(dup[2 * j]), int(dup[2 * j + 1])) for j in range(d)]


def row_shards(g: Csr, n_shards: int) -> np.ndarray:
    """gqc_row_shards: bounds[0..n_shards] of the cost-balanced row blocks."""
    out = np.zeros(n_shards + 1, dtype=np.int32)
    cs = g.c_struct()
    _check(_lib.gqc_row_shards(C.byref(cs), int(n_shards), _ptr(out)))
    return out


def cluster_sweep_multi(g: Csr, sigmas: Sequence[float], devices: Sequence[int], want_v: bool = False,
                        want_succ: bool = False, want_center: bool = True, want_intra: bool = False):
    """gqc_cluster_sweep_multi: the sweep row-sharded over `devices` (one
    shard per entry; repeats put several shards on one device). Returns
    (assignments, v, succ, intra) like cluster_sweep."""
    s = np.ascontiguousarray(np.atleast_1d(np.asarray(sigmas, dtype=np.float64)))
    d = np.ascontiguousarray(np.asarray(devices, dtype=np.int32))
    S, n = len(s), g.n
    v = np.empty((S, n)) if want_v else None
    succ = np.empty((S, n), dtype=np.int32) if want_succ else None
    center = np.empty((S, n), dtype=np.int32) if want_center else None
    intra = np.zeros(S, dtype=np.int64) if want_intra else None
    ci = np.empty((S, n), dtype=np.int32)
    k = np.zeros(S, dtype=np.int32)
    cs = g.c_struct()
    _check(_lib.gqc_cluster_sweep_multi(C.byref(cs), _ptr(s), S, _ptr(d), len(d), _ptr(v), _ptr(succ),
                                        _ptr(center), _ptr(ci), _ptr(k), _ptr(intra)))
    if center is None:
        out = [ClusterAssignment(None, ci[q], int(k[q]), centers=np.zeros(0, np.int32)) for q in range(S)]
    else:
        out = [ClusterAssignment(center[q], ci[q], int(k[q])) for q in range(S)]
    return out, v, succ, intra


def potentials_multi(g: Csr, sigmas: Sequence[float], devices: Sequence[int]) -> np.ndarray:
    s = np.ascontiguousarray(np.atleast_1d(np.asarray(sigmas, dtype=np.float64)))
    d = np.ascontiguousarray(np.asarray(devices, dtype=np.int32))
    out = np.empty((len(s), g.n), dtype=np.float64)
    cs = g.c_struct()
    _check(_lib.gqc_potentials_multi(C.byref(cs), _ptr(s), len(s), _ptr(d), len(d), _ptr(out)))
    return out


def cluster(g: Csr, sigma: float, workers: int = 1) -> ClusterAssignment:
    if not (sigma > 0.0):
        raise ValueError("sigma must be positive")
    if workers < 1:
        raise ValueError("workers must be at least 1")
    res, _, _ = cluster_sweep(g, [sigma])
    return res[0]


# ---------------------------------------------------------------- device API
class DeviceCsr:
    """A CSR resident in device memory (torch tensors as the allocator)."""

    def __init__(self, g: Csr, device="cuda"):
        import torch
        self.n, self.nnz, self.W = g.n, g.nnz, float(g.W)
        self.offsets = torch.from_numpy(g.offsets).to(device)
        self.nbr = torch.from_numpy(g.nbr if g.nnz else np.zeros(1, np.int32)).to(device)
        unit = g.w is None or bool(np.all(g.w == 1.0))
        self.w = None if unit else torch.from_numpy(g.w).to(device)

    def c_struct(self) -> _GqcCsr:
        return _GqcCsr(self.n, self.nnz, self.offsets.data_ptr(), self.nbr.data_ptr(),
                       None if self.w is None else self.w.data_ptr(), self.W)


def dev_potentials(dg: DeviceCsr, sigmas, row_begin: int, row_end: int, out, stream=None):
    """V rows [row_begin, row_end) node-major into the device tensor `out`
    (shape [row_end-row_begin, S], float64) on `stream` (torch stream)."""
    s = np.ascontiguousarray(np.atleast_1d(np.asarray(sigmas, dtype=np.float64)))
    cs = dg.c_struct()
    sp = None if stream is None else C.c_void_p(stream.cuda_stream)
    _check(_lib.gqc_dev_potentials(C.byref(cs), _ptr(s), len(s), int(row_begin), int(row_end),
                                   C.c_void_p(out.data_ptr()), sp))


def dev_potentials_packed(dg: DeviceCsr, sigmas, row_begin: int, row_end: int, out, chunk: int, chunk_stride: int,
                          stream=None):
    """V rows [row_begin, row_end) packed in sigma chunks: sigma k of row i at
    out.flat[(k // chunk) * chunk_stride + (i - row_begin) * chunk + k % chunk]
    (float64 device tensor), the send layout of the sigma-sharded exchange."""
    s = np.ascontiguousarray(np.atleast_1d(np.asarray(sigmas, dtype=np.float64)))
    cs = dg.c_struct()
    sp = None if stream is None else C.c_void_p(stream.cuda_stream)
    _check(_lib.gqc_dev_potentials_packed(C.byref(cs), _ptr(s), len(s), int(row_begin), int(row_end),
                                          C.c_void_p(out.data_ptr()), int(chunk), int(chunk_stride), sp))


def dev_potentials_peer(dg: DeviceCsr, sigmas, row_begin: int, row_end: int, chunk_ptrs, chunk: int, stream=None):
    """gqc_dev_potentials_peer: sigma chunk q of rows [row_begin, row_end) to
    chunk_ptrs[q] + ((i - row_begin) * chunk + k % chunk) * 8 (raw device
    addresses: local, peer or IPC-mapped)."""
    s = np.ascontiguousarray(np.atleast_1d(np.asarray(sigmas, dtype=np.float64)))
    ptrs = (C.c_void_p * len(chunk_ptrs))(*[int(p) for p in chunk_ptrs])
    cs = dg.c_struct()
    sp = None if stream is None else C.c_void_p(stream.cuda_stream)
    _check(_lib.gqc_dev_potentials_peer(C.byref(cs), _ptr(s), len(s), int(row_begin), int(row_end), ptrs,
                                        len(chunk_ptrs), int(chunk), sp))


IPC_HANDLE_BYTES = 64


class IpcBuffer:
    """Device memory another process can map (gqc_ipc_alloc), exposed to torch
    through __cuda_array_interface__ (zero copy)."""

    def __init__(self, nbytes: int):
        p = C.c_void_p()
        self.handle = C.create_string_buffer(IPC_HANDLE_BYTES)
        _check(_lib.gqc_ipc_alloc(int(nbytes), C.byref(p), self.handle))
        self.ptr = int(p.value)
        self.nbytes = int(nbytes)

    def handle_bytes(self) -> bytes:
        return self.handle.raw

    def as_tensor(self, dtype, shape, device):
        import torch
        itemsize = torch.empty((), dtype=dtype).element_size()
        typestr = {torch.float64: "<f8", torch.int32: "<i4", torch.float32: "<f4"}[dtype]
        holder = type("CudaArray", (), {})()
        holder.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (self.ptr, False),
                                           "version": 2, "strides": None}
        assert int(np.prod(shape)) * itemsize <= self.nbytes
        return torch.as_tensor(holder, device=device)

    def free(self):
        if self.ptr:
            _check(_lib.gqc_ipc_free(C.c_void_p(self.ptr)))
            self.ptr = 0


def ipc_open(handle: bytes) -> int:
    """Map another process's gqc_ipc_alloc buffer on GQC_OPT_DEVICE; returns its address here."""
    p = C.c_void_p()
    buf = C.create_string_buffer(bytes(handle), IPC_HANDLE_BYTES)
    _check(_lib.gqc_ipc_open(buf, C.byref(p)))
    return int(p.value)


def ipc_close(ptr: int):
    _check(_lib.gqc_ipc_close(C.c_void_p(int(ptr))))


def dev_ggd_workspace(n: int, n_sigma: int) -> int:
    return int(_lib.gqc_dev_ggd_workspace(n, n_sigma))


def dev_ggd(dg: DeviceCsr, v, n_sigma: int, succ, center, cluster_index, num_clusters, workspace, stream=None):
    cs = dg.c_struct()
    sp = None if stream is None else C.c_void_p(stream.cuda_stream)
    p = lambda t: None if t is None else C.c_void_p(t.data_ptr())
    _check(_lib.gqc_dev_ggd(C.byref(cs), p(v), int(n_sigma), p(succ), p(center), p(cluster_index),
                            p(num_clusters), p(workspace), workspace.numel() * workspace.element_size(), sp))


def dev_transpose(v_nm, n: int, n_sigma: int, v_sm, stream=None):
    sp = None if stream is None else C.c_void_p(stream.cuda_stream)
    _check(_lib.gqc_dev_transpose(C.c_void_p(v_nm.data_ptr()), n, n_sigma, C.c_void_p(v_sm.data_ptr()), sp))


def dev_successors(dg: DeviceCsr, v, n_sigma: int, row_begin: int, row_end: int, succ_rows, stream=None):
    """GGD argmin of rows [row_begin, row_end) from the full node-major V,
    node-major into succ_rows[(i - row_begin), k] (int32 device tensor)."""
    cs = dg.c_struct()
    sp = None if stream is None else C.c_void_p(stream.cuda_stream)
    _check(_lib.gqc_dev_successors(C.byref(cs), C.c_void_p(v.data_ptr()), int(n_sigma), int(row_begin), int(row_end),
                                   C.c_void_p(succ_rows.data_ptr()), sp))


def dev_resolve_workspace(n: int, n_sigma: int) -> int:
    return int(_lib.gqc_dev_resolve_workspace(n, n_sigma))


def dev_resolve(n: int, n_sigma: int, succ_nm, center, cluster_index, num_clusters, workspace, stream=None):
    """Centers / dense cluster indices (sigma-major) and counts from a
    node-major successor matrix [n, n_sigma]."""
    sp = None if stream is None else C.c_void_p(stream.cuda_stream)
    p = lambda t: C.c_void_p(t.data_ptr())
    _check(_lib.gqc_dev_resolve(int(n), int(n_sigma), p(succ_nm), p(center), p(cluster_index), p(num_clusters),
                                p(workspace), workspace.numel() * workspace.element_size(), sp))
