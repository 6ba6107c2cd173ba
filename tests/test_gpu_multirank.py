"""Multi-GPU partition on one GPU: two ranks (two processes
sharing cuda:0, gloo) run the layer step with every MatMul sharded by BSGS baby-step window --
partial accumulators, one exact all-reduce, finish + mask at each output's owner, all-gathers of
the ciphertexts a later MatMul consumes whole -- and the gathered masked outputs and server
shares are bit-identical to the one-rank step (which test_gpu_layer pins against the oracle)."""
import os
import pickle
import socket
import tempfile

import numpy as np
import pytest
import torch

import blb_inputs as bi

pytestmark = pytest.mark.gpu

blb = pytest.importorskip("paper_2508_19525_b200")

L, D, H, FFN = 32, 64, 4, 128
BSGS = {"qkv": 8, "oproj": 4, "ffn1": 8, "ffn2": 4, "qk": 0}
SEQ = 9


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def build(rank: int, world: int):
    from paper_2508_19525_b200 import packing
    from paper_2508_19525_b200.layer import Dims, FusedLinearLayer
    params = blb.Params.from_preset(bi.QKTOY)
    layer = FusedLinearLayer(params, Dims(L, D, H, FFN), rank, world, bsgs=BSGS)
    rng = np.random.default_rng(7)
    W = [rng.normal(0.0, 0.04, s) for s in ((D, D), (D, D), (D, D), (D, D), (D, FFN), (FFN, D))]
    keys, sk = blb.keygen(params, bi.crypto_key(4, 78), layer.rotation_steps(), relin=True)
    layer.load_weights(*W)
    S = bi.softmax_rows(rng.normal(0.0, 1.0, (H, L, L)))
    V = rng.normal(0.0, 1.0, (H, L, D // H))
    sv_s, sv_v = packing.softmax_v_operands(S, V, params.n)
    slots = {"qkv": packing.spatial_slots(rng.normal(0, 1, (L, D)), params.n), "sv_s": sv_s, "sv_v": sv_v,
             "ffn1": packing.spatial_slots(rng.normal(0, 1, (L, D)), params.n),
             "ffn2": packing.spatial_slots(rng.normal(0, 1, (L, FFN)), params.n)}
    delta = 2.0 ** bi.QKTOY.log_delta
    inputs, cid = {}, 0
    for name, zs in slots.items():
        pts = params.encode(torch.tensor(zs), delta, layer.level)
        inputs[name] = []
        for b in range(zs.shape[0]):
            inputs[name].append(blb.encrypt(params, sk, pts[b], layer.level, bi.crypto_key(5, 78), 300 + cid, delta))
            cid += 1
    return params, layer, keys, inputs


def run_step(layer, keys, inputs):
    """-> {block: (first id, [masked u64 arrays], [share u64 arrays])} gathered over the ranks."""
    import torch.distributed as dist
    from paper_2508_19525_b200.layer import allgather_ragged
    res = layer.step(keys, inputs, bi.crypto_key(3, 78), seq=SEQ)
    out = {}
    world = layer.world
    by_name = {name: (id0, m, s) for name, id0, (m, s) in res}
    for name in ("qk", "qkv", "oproj", "ffn1", "ffn2"):
        id0, m, s = by_name.get(name, (None, None, None))
        items = [] if m is None else [torch.cat([m[t].reshape(-1), s[t].reshape(-1)]).cpu() for t in range(m.shape[0])]
        if world > 1:
            N = layer.p.N
            items = allgather_ragged(items, layer.mask_counts(name), like=torch.empty(3 * N, dtype=torch.int64))
            ids = [None] * world
            dist.all_gather_object(ids, id0)
            id0 = min(i for i in ids if i is not None)
        out[name] = (id0, [blb.to_numpy_u64(x) for x in items])
    return out


def worker(rank: int, world: int, port: int, path: str):
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank, world_size=world)
    try:
        params, layer, keys, inputs = build(rank, world)
        out = run_step(layer, keys, inputs)
        if rank == 0:
            with open(path, "wb") as f:
                pickle.dump(out, f)
    finally:
        dist.destroy_process_group()


def test_two_ranks_bit_identical_to_one_rank():
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "r2.pkl")
        mp.spawn(worker, args=(2, free_port(), path), nprocs=2, join=True)
        with open(path, "rb") as f:
            got = pickle.load(f)
    params, layer, keys, inputs = build(0, 1)
    ref = run_step(layer, keys, inputs)
    assert sorted(got) == sorted(ref)
    for name in ref:
        assert got[name][0] == ref[name][0], name
        assert len(got[name][1]) == len(ref[name][1]) > 0, name
        for a, b in zip(got[name][1], ref[name][1]):
            assert np.array_equal(a, b), name


@pytest.mark.parametrize("world", [2, 3])
def test_window_plans_sum_to_the_whole_plan(world):
    """ct-pt and ct-ct windows partition [0, B): per-window accumulators summed (exact u64) and
    finished equal the single-call outputs, limb for limb (no process group needed)."""
    from paper_2508_19525_b200.layer import shard
    params = blb.Params.from_preset(bi.QKTOY)
    rng = np.random.default_rng(world)
    Lq, d, Hq = 32, 64, 4
    Wm = rng.normal(0, 0.05, (d, 96))
    full = blb.MatmulPlan(params, Lq, d, 96, bsgs_B=8, level=4)
    keys, sk = blb.keygen(params, bi.crypto_key(4, 79), full.rotation_steps(), relin=True)
    from paper_2508_19525_b200 import packing
    zs = packing.spatial_slots(rng.normal(0, 1, (Lq, d)), params.n)
    delta = 2.0 ** 40
    cts = [blb.encrypt(params, sk, params.encode(torch.tensor(z), delta, 4), 4, bi.crypto_key(5, 79), 10 + b, delta)
           for b, z in enumerate(zs)]
    ref = full(keys, cts, full.encode_weights(Wm))
    acc = None
    for r in range(world):
        pl = blb.MatmulPlan(params, Lq, d, 96, bsgs_B=8, level=4, window=shard(full.B, r, world))
        a = pl.acc(keys, cts, pl.encode_weights(Wm))
        acc = a if acc is None else acc + a   # int64 wrap-around add = u64 add
    got = pl.finish(keys, acc, 0, full.n_out, cts[0].scale)
    for x, y in zip(got, ref):
        assert x.scale == y.scale and torch.equal(x.data, y.data)
    # ct-ct Q K^T (reading C13)
    qk = blb.QKPlan(params, Lq, Hq, 32, level=3)
    keys2, sk2 = blb.keygen(params, bi.crypto_key(4, 80), qk.rotation_steps(), relin=True)
    Q = [blb.encrypt(params, sk2, params.encode(torch.tensor(rng.uniform(-1, 1, params.n)), delta, 3), 3,
                     bi.crypto_key(5, 80), 40 + j, delta) for j in range(qk.J)]
    K = [blb.encrypt(params, sk2, params.encode(torch.tensor(rng.uniform(-1, 1, params.n)), delta, 3), 3,
                     bi.crypto_key(5, 80), 60 + j, delta) for j in range(qk.J)]
    ref = qk(keys2, Q, K, qk.encode_masks())
    acc = None
    for r in range(world):
        pw = blb.QKPlan(params, Lq, Hq, 32, level=3, window=shard(qk.B, r, world))
        a = pw.acc(keys2, Q, K, pw.encode_masks())
        acc = a if acc is None else acc + a
    a0, na = pw.acc_range(0, qk.n_out)
    got = pw.finish(keys2, acc, 0, qk.n_out, Q[0].scale, K[0].scale)
    for x, y in zip(got, ref):
        assert x.scale == y.scale and torch.equal(x.data, y.data)
    # an output slice finishes from its own accumulator slots
    o0, cnt = shard(qk.n_out, 1, 2)
    a0, na = pw.acc_range(o0, cnt)
    per = pw.acc_numel() // pw.acc_range(0, qk.n_out)[1]
    part = pw.finish(keys2, acc[a0 * per:(a0 + na) * per].contiguous(), o0, cnt, Q[0].scale, K[0].scale)
    for x, y in zip(part, ref[o0:o0 + cnt]):
        assert torch.equal(x.data, y.data)
