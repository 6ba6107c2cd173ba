"""The layer step and its serving pipeline (layer.LayerPipeline, the e2e path of bench.py) on a
small ring with the BERT chain shape: the pipelined host-to-host run (copy stream, double-buffered
device inputs, pinned outputs) returns exactly the masked outputs and server shares of a plain
FusedLinearLayer.step on device-resident inputs, for several steps in flight."""
import numpy as np
import pytest
import torch

import blb_inputs as bi

pytestmark = pytest.mark.gpu

blb = pytest.importorskip("paper_2508_19525_b200")
from paper_2508_19525_b200 import packing  # noqa: E402
from paper_2508_19525_b200.layer import Dims, FusedLinearLayer, LayerPipeline  # noqa: E402


def flat(res):
    out = []
    for _, _, r in res:
        out.extend(r if isinstance(r, (tuple, list)) else (r,))
    return out


def test_layer_pipeline_matches_step():
    P = bi.QKTOY
    params = blb.Params.from_preset(P)
    L, d, H, ffn = 32, 64, 4, 128
    layer = FusedLinearLayer(params, Dims(L, d, H, ffn), bsgs={"qkv": 8, "oproj": 4, "ffn1": 8, "ffn2": 4})
    rng = np.random.default_rng(7)
    W = lambda r, c: rng.normal(0.0, 0.04, (r, c))  # noqa: E731
    keys, sk = blb.keygen(params, bi.crypto_key(4, 77), layer.rotation_steps(), relin=True)
    layer.load_weights(W(d, d), W(d, d), W(d, d), W(d, d), W(d, ffn), W(ffn, d))
    S = bi.softmax_rows(rng.normal(0.0, 1.0, (H, L, L)))
    V = rng.normal(0.0, 1.0, (H, L, d // H))
    sv_s, sv_v = packing.softmax_v_operands(S, V, params.n)
    slots = {"qkv": packing.spatial_slots(rng.normal(0, 1, (L, d)), params.n), "sv_s": sv_s, "sv_v": sv_v,
             "ffn1": packing.spatial_slots(rng.normal(0, 1, (L, d)), params.n),
             "ffn2": packing.spatial_slots(rng.normal(0, 1, (L, ffn)), params.n)}
    delta = 2.0 ** P.log_delta
    inputs, cid = {}, 0
    for name, zs in slots.items():
        pts = params.encode(torch.tensor(zs), delta, layer.level)
        inputs[name] = []
        for b in range(zs.shape[0]):
            inputs[name].append(blb.encrypt(params, sk, pts[b], layer.level, bi.crypto_key(5, 77), 100 + cid, delta))
            cid += 1
    mask_key = bi.crypto_key(3, 77)
    ref = [t.cpu() for t in flat(layer.step(keys, inputs, mask_key))]
    assert ref and all(t.numel() for t in ref)
    host_in = {k: [c.data.cpu().pin_memory() for c in v] for k, v in inputs.items()}
    pipe = LayerPipeline(layer, keys, mask_key, inputs)
    outs = [pipe.submit(host_in) for _ in range(3)]  # three steps in flight, two buffer sets
    pipe.drain()
    torch.cuda.synchronize()
    for got in (outs[1], outs[2]):
        assert len(got) == len(ref)
        for a, b in zip(got, ref):
            assert torch.equal(a, b)
