"""The multi-process fused exchange (PeerSigmaShardedSweep +
gqc_dev_potentials_peer + CUDA IPC): each rank's potential kernel stores
sigma chunk q of its rows straight into rank q's receive buffer, mapped from
another process. Run here as 2 and 3 processes on ONE GPU (CUDA IPC between
processes of the same device; gloo barrier after a device sync: no kernel
waits on another), each rank's V chunk and labels compared bit for bit with
the single-process sweep, over two steps (alternating receive buffers)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path, balanced):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_14641_b200 import native as N
        from paper_2305_14641_b200 import sharded
        from paper_2305_14641_b200.sweep import log_sigma_grid
        from tests import helpers as H
        torch.cuda.set_device(0)
        N.set_device(0)
        off, nbr = H.sbm_csr()
        n = len(off) - 1
        sig = np.ascontiguousarray(log_sigma_grid(10.0, 32))
        S = len(sig)
        csr = N.Csr(off, nbr, None, 10.0)
        dg = N.DeviceCsr(csr, torch.device("cuda", 0))
        stream = torch.cuda.Stream()
        chunk = sharded.sigma_chunk(S, world)
        center = torch.empty((chunk, n), dtype=torch.int32, device="cuda")
        ws = torch.empty(N.dev_ggd_workspace(n, chunk), dtype=torch.uint8, device="cuda")
        bounds = [int(b) for b in N.row_shards(csr, world)] if balanced else None

        def pot(b, e, ptrs, ch):
            N.dev_potentials_peer(dg, sig, b, e, ptrs, ch, stream)

        def ggd(v, ci, nc):
            N.dev_ggd(dg, v, chunk, None, center, ci, nc, ws, stream)

        with torch.cuda.stream(stream):
            sw = sharded.PeerSigmaShardedSweep(n, S, rank, world, "cuda", pot, ggd, bounds=bounds)
        res, v_ref, _ = N.cluster_sweep(csr, sig, want_v=True)
        ok = True
        for step in range(2):
            with torch.cuda.stream(stream):
                sw.potentials()
                v = sw.exchange()
                sw.ggd(v)
            torch.cuda.synchronize()
            for q in range(sw.s_begin, sw.s_end):
                col = q - sw.s_begin
                got = v[:, col].cpu().numpy()
                ok &= np.array_equal(got.view(np.int64), v_ref[q].view(np.int64))
                ok &= np.array_equal(sw.ci[col].cpu().numpy(), res[q].cluster_index)
                ok &= int(sw.nc[col]) == res[q].num_clusters
            dist.barrier()
        sw.close()
        with open(f"{out_path}.{rank}", "w") as f:
            f.write("ok" if ok else "mismatch")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,balanced", [(2, False), (3, True)])
def test_peer_exchange_between_processes(world, balanced, tmp_path):
    out = tmp_path / "r"
    mp.start_processes(_worker, args=(world, _free_port(), str(out), balanced), nprocs=world, join=True,
                       start_method="spawn")
    for r in range(world):
        assert (tmp_path / f"r.{r}").read_text() == "ok"
