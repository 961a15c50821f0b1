"""Row-sharded sweep over several GPUs (one process per GPU, torch.distributed).

The potential of row i depends only on row i of the CSR (potential.cpp:18-37),
so the sweep shards by rows with the full CSR replicated on every rank and no
communication while it runs. GGD needs every neighbour's potential
(ggd.cpp:7-24), which is the one real exchange step: a single all-gather of V
(fp64, node-major [rows][n_sigma]) over NVLink, after which every rank runs
GGD on the full field, so labels are identical on all ranks without a second
collective.

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
