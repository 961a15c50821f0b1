"""Multi-rank host path on CPU (gloo, world_size 2 and 3): row partition,
equal-slab all-gather, and assembly reproduce the single-process field bit
for bit when each rank computes only its rows (the oracle stands in for the
device kernel here; on the GPU the same callable wraps gqc_dev_potentials)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2305_14641_b200 import sharded


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_row_shards_partition_rows():
    for n in (1, 2, 7, 34, 1000, 1_000_003):
        for world in (1, 2, 3, 4, 8):
            got = [sharded.row_shard(n, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == n
            for (a, b), (c, d) in zip(got[:-1], got[1:]):
                assert b == c and a <= b
            assert all(b - a <= sharded.row_block(n, world) for a, b in got)


def _worker(rank, world, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle as O
        from tests import helpers as H
        g = H.random_graph(101, 4.0, seed=11, unit=True)
        sig = [0.7, 2.3, 5.0]

        def compute_rows(begin, end, out):
            rows = np.arange(begin, end, dtype=np.int32)
            for q, s in enumerate(sig):
                out[:, q] = torch.from_numpy(O.potentials_rows(g.offsets, g.nbr, g.wt, 10.0, s, rows))

        full = sharded.sharded_field(g.n, len(sig), compute_rows, rank, world, "cpu")
        if rank == 0:
            ref = np.stack([O.potentials(g.offsets, g.nbr, g.wt, 10.0, s) for s in sig], axis=1)
            ok = np.array_equal(full.numpy().view(np.int64), ref.view(np.int64))
            with open(result_path, "w") as f:
                f.write("ok" if ok else "mismatch")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_field_matches_single_process(world, tmp_path):
    result = tmp_path / "result.txt"
    mp.start_processes(_worker, args=(world, _free_port(), str(result)), nprocs=world, join=True,
                       start_method="spawn")
    assert result.read_text() == "ok"


def _worker_ggd(rank, world, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle as O
        from tests import helpers as H
        g = H.random_graph(97, 3.0, seed=12, unit=True)
        sig = [0.7, 2.3, 5.0, 30.0]

        def potentials_rows(begin, end, out):
            rows = np.arange(begin, end, dtype=np.int32)
            for q, s in enumerate(sig):
                out[:, q] = torch.from_numpy(O.potentials_rows(g.offsets, g.nbr, g.wt, 10.0, s, rows))

        def successors_rows(V, begin, end, out):
            for q in range(len(sig)):
                full = O.build_successors(g.offsets, g.nbr, V[:, q].numpy().copy())
                out[:, q] = torch.from_numpy(full[begin:end])

        def resolve(succ):
            res = [O.resolve_centers(succ[:, q].numpy().copy()) for q in range(len(sig))]
            return res

        sweep = sharded.ShardedSweep(g.n, len(sig), rank, world, "cpu", potentials_rows, successors_rows, resolve)
        V, succ, res = sweep.step()
        ok = True
        for q, s in enumerate(sig):
            v, so, co, cio, ko = O.cluster(g.offsets, g.nbr, g.wt, 10.0, s)
            ok &= np.array_equal(V[:, q].numpy().view(np.int64), v.view(np.int64))
            ok &= np.array_equal(succ[:, q].numpy(), so)
            ok &= np.array_equal(res[q][0], co) and np.array_equal(res[q][1], cio) and res[q][2] == ko
        with open(f"{result_path}.{rank}", "w") as f:
            f.write("ok" if ok else "mismatch")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_ggd_matches_single_process(world, tmp_path):
    # the multi-GPU schedule with the GGD argmin sharded: every rank ends with
    # the single-process labels
    result = tmp_path / "r"
    mp.start_processes(_worker_ggd, args=(world, _free_port(), str(result)), nprocs=world, join=True,
                       start_method="spawn")
    for r in range(world):
        assert (tmp_path / f"r.{r}").read_text() == "ok"


def test_sigma_shards_partition_the_grid():
    for S in (1, 3, 7, 32, 33):
        for world in (1, 2, 3, 4, 8):
            got = [sharded.sigma_shard(S, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == S
            for (a, b), (c, d) in zip(got[:-1], got[1:]):
                assert b == c and a <= b
            assert all(b - a <= sharded.sigma_chunk(S, world) for a, b in got)


def _worker_sigma(rank, world, port, result_path, n_nodes, sig, bounds=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle as O
        from tests import helpers as H
        g = H.random_graph(n_nodes, 3.0, seed=13, unit=True)
        S = len(sig)

        def potentials_packed(begin, end, send, chunk, stride):
            rows = np.arange(begin, end, dtype=np.int32)
            for k, s in enumerate(sig):
                q, r = divmod(k, chunk)
                v = torch.from_numpy(O.potentials_rows(g.offsets, g.nbr, g.wt, 10.0, s, rows))
                send[q * stride + r: q * stride + r + (end - begin) * chunk: chunk] = v

        def ggd(V, ci, nc):
            for k in range(V.shape[1]):
                succ = O.build_successors(g.offsets, g.nbr, V[:, k].numpy().copy())
                _, cik, kk = O.resolve_centers(succ)
                ci[k] = torch.from_numpy(cik)
                nc[k] = kk

        if bounds == "cost":  # gqc_row_shards (host-only call): degree-balanced blocks
            from paper_2305_14641_b200 import native as N
            b = [int(x) for x in N.row_shards(N.Csr(g.offsets, g.nbr, None, 10.0), world)]
        else:
            b = bounds
        sweep = sharded.SigmaShardedSweep(g.n, S, rank, world, "cpu", potentials_packed, ggd, bounds=b)
        ci, nc = sweep.step()
        ok = tuple(ci.shape) == (S, g.n) and tuple(nc.shape) == (S,)
        ref = [O.cluster(g.offsets, g.nbr, g.wt, 10.0, s) for s in sig]
        for q in range(S):
            ok &= np.array_equal(ci[q].numpy(), ref[q][3]) and int(nc[q]) == ref[q][4]
        # sharded label layout (bench default): counts on every rank, each
        # rank's own sigma chunk of labels in sweep.ci
        sweep.potentials()
        sweep.ggd(sweep.exchange())
        nc2 = sweep.gather_counts()
        ok &= [int(x) for x in nc2] == [r[4] for r in ref]
        for q in range(sweep.s_begin, sweep.s_end):
            ok &= np.array_equal(sweep.ci[q - sweep.s_begin].numpy(), ref[q][3])
        with open(f"{result_path}.{rank}", "w") as f:
            f.write("ok" if ok else "mismatch")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_nodes,sig", [(2, 97, [0.7, 2.3, 5.0, 30.0]),
                                               (3, 101, [0.7, 2.3, 5.0, 9.0, 30.0]),  # padded sigma chunk
                                               (3, 2, [1.0, 4.0]),                     # fewer rows / sigmas than ranks
                                               (2, 64, [3.0])])                        # one rank with no sigma
def test_gloo_sigma_sharded_ggd_matches_single_process(world, n_nodes, sig, tmp_path):
    # the production multi-GPU schedule: row-sharded potentials -> all-to-all of
    # V by sigma chunk -> per-chunk GGD -> all-gather labels; every rank ends
    # with the single-process labels of every sigma
    result = tmp_path / "r"
    mp.start_processes(_worker_sigma, args=(world, _free_port(), str(result), n_nodes, sig), nprocs=world,
                       join=True, start_method="spawn")
    for r in range(world):
        assert (tmp_path / f"r.{r}").read_text() == "ok"


@pytest.mark.parametrize("world,n_nodes,sig,bounds", [(2, 97, [0.7, 2.3, 5.0, 30.0], "cost"),
                                                      (3, 101, [0.7, 2.3, 5.0, 9.0, 30.0], "cost"),
                                                      (2, 97, [0.7, 2.3, 30.0], [0, 11, 97]),
                                                      (3, 80, [1.0, 4.0, 9.0], [0, 0, 70, 80])])  # an empty rank
def test_gloo_sigma_sharded_uneven_row_blocks(world, n_nodes, sig, bounds, tmp_path):
    # cost-balanced (gqc_row_shards) or arbitrary uneven row blocks: the
    # all-to-all with per-rank split sizes still lands every chunk's rows in
    # order, and every rank ends with the single-process labels
    result = tmp_path / "r"
    mp.start_processes(_worker_sigma, args=(world, _free_port(), str(result), n_nodes, sig, bounds), nprocs=world,
                       join=True, start_method="spawn")
    for r in range(world):
        assert (tmp_path / f"r.{r}").read_text() == "ok"
