"""Sharded sweep over several GPUs (one process per GPU, torch.distributed).

The potential of row i depends only on row i of the CSR (potential.cpp:18-37),
so the sweep shards by rows with the full CSR replicated on every rank and no
communication while it runs. GGD needs every neighbour's potential
(ggd.cpp:7-24), which is the one real exchange step: a single all-gather of V
(fp64, node-major [rows][n_sigma]) over NVLink, after which every rank runs
GGD on the full field, so labels are identical on all ranks without a second
collective.

SigmaShardedSweep is the production schedule: potentials stay row-sharded,
but the exchange hands every rank the full rows of its own sigma chunk (one
all-to-all of V, 1/world of the all-gather's bytes), GGD then runs on that
chunk only (every sigma's GGD is independent, ggd.cpp:7-57), and one
all-gather assembles the labels. ShardedSweep (all-gather V, row-sharded
successors, replicated resolve) is kept as the simpler schedule.

The host logic here is device-agnostic (it takes the compute step as a
callable) so the partition/gather/assembly path is tested on CPU with gloo.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist


def row_block(n: int, world: int) -> int:
    """Rows per rank (the last rank's block is padded)."""
    return (n + world - 1) // world


def row_shard(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Rank `rank` owns rows [begin, end): equal blocks of ceil(n/world) so
    that every rank contributes an equal-sized slab to the all-gather."""
    b = row_block(n, world)
    begin = min(n, rank * b)
    end = min(n, begin + b)
    return begin, end


def gather_rows(shard: torch.Tensor, n: int, group=None, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """All-gather equal [block, S] slabs into the full [n, S] field.
    `shard` must have row_block(n, world) rows (padding rows are ignored)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return shard[:n]
    block = shard.shape[0]
    if out is None:
        out = torch.empty((world * block,) + tuple(shard.shape[1:]), dtype=shard.dtype, device=shard.device)
    dist.all_gather_into_tensor(out, shard.contiguous(), group=group)
    return out[:n]


def sharded_field(n: int, n_sigma: int, compute_rows: Callable[[int, int, torch.Tensor], None], rank: int,
                  world: int, device, group=None, dtype=torch.float64, shard_buf=None, full_buf=None):
    """Compute this rank's rows with compute_rows(begin, end, out[:end-begin])
    and all-gather the field. Returns the full [n, n_sigma] tensor."""
    block = row_block(n, world)
    begin, end = row_shard(n, world, rank)
    shard = shard_buf if shard_buf is not None else torch.zeros((block, n_sigma), dtype=dtype, device=device)
    if end > begin:
        compute_rows(begin, end, shard[: end - begin])
    return gather_rows(shard, n, group, full_buf)


class ShardedSweep:
    """One multi-GPU step of the sweep with the GGD argmin sharded too:

        potentials of own rows -> all-gather V (fp64) ->
        successors of own rows -> all-gather succ (int32) -> centers/labels

    Every collective is an equal-slab all-gather of node-major rows. The
    device operations are injected (native gqc_dev_* on the GPU; the oracle in
    the CPU gloo tests), so this class is the whole host-side schedule.

      potentials_rows(begin, end, out[rows, S])
      successors_rows(V[n, S], begin, end, out[rows, S] int32)
      resolve(succ[n, S] int32) -> (center [S, n], cluster_index [S, n], num_clusters [S])
    """

    def __init__(self, n, n_sigma, rank, world, device, potentials_rows, successors_rows, resolve, group=None):
        self.n, self.S, self.rank, self.world, self.group = n, n_sigma, rank, world, group
        self.block = row_block(n, world)
        self.begin, self.end = row_shard(n, world, rank)
        self.potentials_rows, self.successors_rows, self.resolve = potentials_rows, successors_rows, resolve
        self.shard_v = torch.zeros((self.block, n_sigma), dtype=torch.float64, device=device)
        self.shard_s = torch.zeros((self.block, n_sigma), dtype=torch.int32, device=device)
        big = world > 1
        self.full_v = torch.empty((world * self.block, n_sigma), dtype=torch.float64, device=device) if big else None
        self.full_s = torch.empty((world * self.block, n_sigma), dtype=torch.int32, device=device) if big else None

    def potentials(self):
        rows = self.end - self.begin
        if rows > 0:
            self.potentials_rows(self.begin, self.end, self.shard_v[:rows])
        return gather_rows(self.shard_v, self.n, self.group, self.full_v)

    def successors(self, V):
        rows = self.end - self.begin
        if rows > 0:
            self.successors_rows(V, self.begin, self.end, self.shard_s[:rows])
        return gather_rows(self.shard_s, self.n, self.group, self.full_s)

    def step(self):
        V = self.potentials()
        succ = self.successors(V)
        return V, succ, self.resolve(succ)


def sigma_chunk(n_sigma: int, world: int) -> int:
    """Sigmas per rank in the sigma-sharded GGD (the last chunks are padded)."""
    return (n_sigma + world - 1) // world


def sigma_shard(n_sigma: int, world: int, rank: int) -> Tuple[int, int]:
    """Rank `rank` labels sigmas [begin, end) of the grid."""
    c = sigma_chunk(n_sigma, world)
    begin = min(n_sigma, rank * c)
    return begin, min(n_sigma, begin + c)


class SigmaShardedSweep:
    """One multi-GPU step with the GGD sharded by sigma:

        potentials of own rows, all sigmas (written packed by sigma chunk) ->
        all-to-all: rank q receives every rank's rows of sigma chunk q ->
        GGD (successors, centers, labels) of sigma chunk q over all rows ->
        all-gather of the labels [S][n] and counts [S]

    Bytes on the wire per rank: (world-1)/world * n*S*8/world for V plus the
    labels gather, against (world-1)/world * n*S*(8+4) for all-gather(V) +
    all-gather(succ); and no rank repeats another's GGD work. Row blocks may
    be uneven (cost-balanced `bounds`): the all-to-all then uses per-rank
    split sizes and lands the chunk's rows in order.

      potentials_packed(begin, end, send, chunk, chunk_stride): V rows
          [begin, end) into the flat send buffer, sigma k of row i at
          (k // chunk) * chunk_stride + (i - begin) * chunk + k % chunk
      ggd(V_chunk [n, chunk] node-major, ci [chunk, n] int32, nc [chunk] int32)
    Padding (rows past n, sigmas past S) stays zero and is dropped.
    """

    def __init__(self, n, n_sigma, rank, world, device, potentials_packed, ggd, group=None, bounds=None):
        self.n, self.S, self.rank, self.world, self.group = n, n_sigma, rank, world, group
        # row blocks: `bounds` (world + 1 ascending row ids, e.g. the
        # cost-balanced gqc_row_shards, so skewed graphs give every rank the
        # same work), else equal blocks of ceil(n / world)
        if bounds is None:
            bounds = [row_shard(n, world, r)[0] for r in range(world)] + [n]
        self.bounds = [int(b) for b in bounds]
        assert len(self.bounds) == world + 1 and self.bounds[0] == 0 and self.bounds[-1] == n
        self.rows_of = [self.bounds[r + 1] - self.bounds[r] for r in range(world)]
        self.begin, self.end = self.bounds[rank], self.bounds[rank + 1]
        self.rows = self.end - self.begin
        self.block = max(self.rows_of)
        self.chunk = sigma_chunk(n_sigma, world)
        self.s_begin, self.s_end = sigma_shard(n_sigma, world, rank)
        self.potentials_packed, self.ggd_op = potentials_packed, ggd
        # send: this rank's rows, packed by sigma chunk ([world][rows][chunk]);
        # recv: every rank's rows of this rank's chunk, in row order = the
        # node-major [n][chunk] field (uneven all-to-all splits)
        self.send = torch.zeros(max(1, world * self.rows * self.chunk), dtype=torch.float64, device=device)
        self.recv = torch.zeros(n * self.chunk, dtype=torch.float64, device=device) if world > 1 else self.send
        self.ci = torch.zeros((self.chunk, n), dtype=torch.int32, device=device)
        self.nc = torch.zeros(self.chunk, dtype=torch.int32, device=device)
        self.ci_full = torch.empty((world * self.chunk, n), dtype=torch.int32, device=device) if world > 1 else self.ci
        self.nc_full = torch.empty(world * self.chunk, dtype=torch.int32, device=device) if world > 1 else self.nc

    def potentials(self):
        if self.rows > 0:
            self.potentials_packed(self.begin, self.end, self.send, self.chunk, self.rows * self.chunk)

    def exchange(self):
        """V of this rank's sigma chunk for all rows, node-major [n, chunk]."""
        if self.world > 1:
            dist.all_to_all_single(self.recv, self.send[: self.world * self.rows * self.chunk],
                                   output_split_sizes=[r * self.chunk for r in self.rows_of],
                                   input_split_sizes=[self.rows * self.chunk] * self.world, group=self.group)
        return self.recv[: self.n * self.chunk].view(self.n, self.chunk)

    def ggd(self, v_chunk):
        self.ggd_op(v_chunk, self.ci, self.nc)

    def gather(self):
        """Labels [S, n] and counts [S] of the whole grid on every rank."""
        if self.world > 1:
            dist.all_gather_into_tensor(self.ci_full, self.ci, group=self.group)
            dist.all_gather_into_tensor(self.nc_full, self.nc, group=self.group)
        return self.ci_full[: self.S], self.nc_full[: self.S]

    def gather_counts(self):
        """Counts [S] of the whole grid on every rank (enough for the sweep's
        mutation interval, sweep.cpp:61-71); the labels stay with the rank
        that owns their sigma chunk (rows [s_begin, s_end) of self.ci)."""
        if self.world > 1:
            dist.all_gather_into_tensor(self.nc_full, self.nc, group=self.group)
        return self.nc_full[: self.S]

    def step(self):
        self.potentials()
        v = self.exchange()
        self.ggd(v)
        return self.gather()


class PeerSigmaShardedSweep:
    """SigmaShardedSweep with the exchange fused into the potential kernel
    (gqc_dev_potentials_peer): every rank maps every other rank's receive
    buffer (CUDA IPC, gqc_ipc_alloc / gqc_ipc_open), and its potential kernel
    stores sigma chunk q of its rows straight into rank q's node-major
    V[n][chunk] over NVLink — no all-to-all and no second copy of V. One
    stream-ordered all-reduce of one float per step (NCCL; with gloo a device
    sync + barrier) orders every rank's stores before any rank's GGD reads its
    chunk; receive buffers alternate between steps, so the next step's stores
    never race the previous step's GGD (a rank passes step k+1's barrier only
    after every rank's step-k GGD, which precedes it on that rank's stream).

      potentials_peer(begin, end, chunk_ptrs, chunk): raw device addresses,
          chunk_ptrs[q] = where row `begin` of sigma chunk q goes
      ggd(V_chunk [n, chunk] node-major, ci [chunk, n] int32, nc [chunk] int32)
    """

    def __init__(self, n, n_sigma, rank, world, device, potentials_peer, ggd, group=None, bounds=None):
        from . import native as N
        self.n, self.S, self.rank, self.world, self.group = n, n_sigma, rank, world, group
        if bounds is None:
            bounds = [row_shard(n, world, r)[0] for r in range(world)] + [n]
        self.bounds = [int(b) for b in bounds]
        self.begin, self.end = self.bounds[rank], self.bounds[rank + 1]
        self.rows = self.end - self.begin
        self.chunk = sigma_chunk(n_sigma, world)
        self.n_chunks = (n_sigma + self.chunk - 1) // self.chunk
        self.s_begin, self.s_end = sigma_shard(n_sigma, world, rank)
        self.potentials_peer, self.ggd_op = potentials_peer, ggd
        nbytes = max(1, n * self.chunk) * 8
        self.bufs = [N.IpcBuffer(nbytes) for _ in range(2)]
        mine = [b.handle_bytes() for b in self.bufs]
        if world > 1:
            allh = [None] * world
            dist.all_gather_object(allh, mine, group=group)
        else:
            allh = [mine]
        self.mapped = []
        self.peer = []  # peer[k][q]: base address of rank q's buffer k in this process
        for k in range(2):
            row = []
            for q in range(world):
                if q == rank:
                    row.append(self.bufs[k].ptr)
                else:
                    a = N.ipc_open(allh[q][k])
                    self.mapped.append(a)
                    row.append(a)
            self.peer.append(row)
        self.views = [b.as_tensor(torch.float64, (n, self.chunk), device) for b in self.bufs]
        self.ci = torch.zeros((self.chunk, n), dtype=torch.int32, device=device)
        self.nc = torch.zeros(self.chunk, dtype=torch.int32, device=device)
        self.nc_full = torch.empty(world * self.chunk, dtype=torch.int32, device=device) if world > 1 else self.nc
        self.ci_full = torch.empty((world * self.chunk, n), dtype=torch.int32, device=device) if world > 1 else self.ci
        self.tick = torch.zeros(1, dtype=torch.float32, device=device)
        self.nccl = world > 1 and dist.get_backend(group) == "nccl"
        self.step_k = 0

    def potentials(self):
        k = self.step_k & 1
        if self.rows > 0:
            ptrs = [self.peer[k][q] + self.begin * self.chunk * 8 for q in range(self.n_chunks)]
            self.potentials_peer(self.begin, self.end, ptrs, self.chunk)

    def exchange(self):
        """Orders every rank's stores before this rank's GGD; returns V[n, chunk]."""
        if self.world > 1:
            if self.nccl:
                dist.all_reduce(self.tick, group=self.group)
            else:
                torch.cuda.synchronize()
                dist.barrier(group=self.group)
        v = self.views[self.step_k & 1]
        self.step_k += 1
        return v

    def ggd(self, v_chunk):
        if self.s_end > self.s_begin:
            self.ggd_op(v_chunk, self.ci, self.nc)

    def gather_counts(self):
        if self.world > 1:
            dist.all_gather_into_tensor(self.nc_full, self.nc, group=self.group)
        return self.nc_full[: self.S]

    def gather(self):
        if self.world > 1:
            dist.all_gather_into_tensor(self.ci_full, self.ci, group=self.group)
            dist.all_gather_into_tensor(self.nc_full, self.nc, group=self.group)
        return self.ci_full[: self.S], self.nc_full[: self.S]

    def step(self):
        self.potentials()
        self.ggd(self.exchange())
        return self.gather()

    def close(self):
        from . import native as N
        torch.cuda.synchronize()
        for a in self.mapped:
            N.ipc_close(a)
        self.mapped = []
        for b in self.bufs:
            b.free()
