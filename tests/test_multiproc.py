"""World-size-2 gloo tests (CPU) of the multi-GPU host logic:
output-ciphertext sharding covers every output exactly once, and the padded
ragged all-gather used at the end of each layer (and for the Q / K operands of
Q K^T) reassembles the rank-ordered list bit-exactly."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_partition():
    from paper_2508_19525_b200.layer import shard
    for n in [1, 3, 8, 11, 12, 37]:
        for world in [1, 2, 3, 4, 8]:
            seen = []
            for r in range(world):
                f, c = shard(n, r, world)
                seen += list(range(f, f + c))
            assert seen == list(range(n))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_2508_19525_b200.layer import allgather_ragged, shard
        ok = True
        for n in [11, 3, 8, 1]:
            counts = [shard(n, r, world)[1] for r in range(world)]
            f, c = shard(n, rank, world)
            local = [torch.full((2, 3, 16), 1000 * g + 7, dtype=torch.int64) + torch.arange(96).view(2, 3, 16)
                     for g in range(f, f + c)]
            full = allgather_ragged(local, counts, like=torch.zeros(2, 3, 16, dtype=torch.int64))
            ref = [torch.full((2, 3, 16), 1000 * g + 7, dtype=torch.int64) + torch.arange(96).view(2, 3, 16)
                   for g in range(n)]
            ok &= len(full) == n and all(torch.equal(a, b) for a, b in zip(full, ref))
        # ragged counts that are not a `shard` split (masked V outputs of QKV)
        counts = [0, 3]
        local = [torch.arange(5) + 10 * t for t in range(counts[rank])]
        full = allgather_ragged(local, counts, like=torch.zeros(5, dtype=torch.int64))
        ok &= [x.tolist() for x in full] == [(torch.arange(5) + 10 * t).tolist() for t in range(3)]
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_allgather_ragged_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=120)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: True, 1: True}
