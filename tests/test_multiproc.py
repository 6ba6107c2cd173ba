"""World-size-2 gloo tests (CPU) of the multi-GPU host logic:
output-ciphertext and baby-step-window sharding cover every index exactly once, the exact
all-reduce of partial accumulators adds residues as u64 (two's-complement int64 wrap-around
gives the u64 bits; 8 residues < 2^61 never exceed 2^64), and the padded ragged all-gather used
for the Q / K operands, the Softmax x V outputs and the end-of-layer results reassembles the
rank-ordered list bit-exactly."""
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
        # exact sum of partial accumulators: residues just below 2^61 on every rank (the int64 sum
        # wraps past 2^63 once 4+ such residues are added; the u64 bits are the exact sum)
        from paper_2508_19525_b200.layer import allreduce_sum_
        big = (1 << 61) - 1 - rank
        t = torch.tensor([big, 5 + rank, (1 << 61) - 7], dtype=torch.int64)
        allreduce_sum_(t)
        exact = [sum((1 << 61) - 1 - r for r in range(world)), sum(5 + r for r in range(world)),
                 world * ((1 << 61) - 7)]
        ok &= [int(v) % (1 << 64) for v in t.tolist()] == [e % (1 << 64) for e in exact]
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


def test_u64_sum_via_int64_wraparound():
    """8 ranks' residues < 2^61 summed in int64 (wrapping past 2^63) give the exact u64 sum."""
    vals = [(1 << 61) - 1 - r for r in range(8)]
    t = torch.zeros(1, dtype=torch.int64)
    for v in vals:
        t += torch.tensor([v], dtype=torch.int64)
    assert int(t.item()) % (1 << 64) == sum(vals) and sum(vals) < (1 << 64)


def test_window_partition_of_baby_steps():
    """The baby-step windows of the ranks partition [0, B) for every plan B at every GPU count."""
    from paper_2508_19525_b200.layer import shard
    for B in [4, 8, 16, 64]:
        for world in [1, 2, 4, 8]:
            if world > B:
                continue
            seen = []
            for r in range(world):
                f, c = shard(B, r, world)
                assert c >= 1
                seen += list(range(f, f + c))
            assert seen == list(range(B))
