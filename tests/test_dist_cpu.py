"""World-size-2 gloo tests of the multi-GPU batch plumbing (CPU only)."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2501_02483_b200.batch import gather_rows, shard_range


def test_shard_range_partitions():
    for P in (0, 1, 7, 64):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                lo, hi = shard_range(P, world, r)
                seen.extend(range(lo, hi))
            assert seen == list(range(P))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, P, width, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(P, world, rank)
    rows = np.array([[float(i)] + [i * 10.0 + c for c in range(width - 1)] for i in range(lo, hi)]).reshape(-1, width)
    out = gather_rows(rows, P, device="cpu")
    q.put((rank, out))
    dist.destroy_process_group()


def test_gather_rows_gloo_world2():
    for P, width in ((5, 1), (64, 4), (1, 3)):
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        ps = [ctx.Process(target=_worker, args=(r, 2, port, P, width, q)) for r in range(2)]
        for p in ps:
            p.start()
        res = [q.get(timeout=120) for _ in ps]
        for p in ps:
            p.join(timeout=60)
        want = np.array([[float(i)] + [i * 10.0 + c for c in range(width - 1)] for i in range(P)]).reshape(P, width)
        for _, out in res:
            assert np.array_equal(out, want)


def _worker_sharded(rank, world, port, P, width, q):
    import torch
    import torch.distributed as dist
    from paper_2501_02483_b200.batch import sharded_rows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calls = []

    def local(lo, hi):
        calls.append((lo, hi))
        return torch.tensor([[float(i)] + [i * 10.0 + c for c in range(width - 1)] for i in range(lo, hi)],
                            dtype=torch.float64).reshape(hi - lo, width)
    out = sharded_rows(P, local, width, device="cpu").numpy()
    q.put((rank, calls, out))
    dist.destroy_process_group()


def test_sharded_rows_gloo_world2():
    """Rank orchestration of the sharded batch (api.logdet_many_sharded):
    each rank computes exactly its contiguous block, one all-gather returns
    every row in problem order on every rank (ranks with no problems too)."""
    for P, width in ((64, 3), (3, 2), (1, 2)):
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        ps = [ctx.Process(target=_worker_sharded, args=(r, 2, port, P, width, q)) for r in range(2)]
        for p in ps:
            p.start()
        res = [q.get(timeout=120) for _ in ps]
        for p in ps:
            p.join(timeout=60)
        want = np.array([[float(i)] + [i * 10.0 + c for c in range(width - 1)] for i in range(P)]).reshape(P, width)
        for rank, calls, out in res:
            lo, hi = shard_range(P, 2, rank)
            assert calls == ([(lo, hi)] if hi > lo else [])
            assert np.array_equal(out, want)
