"""The layer step (layer.FusedLinearLayer, what bench.py times) and its serving pipeline
(layer.LayerPipeline, the e2e path of bench.py) on a small ring with the BERT chain shape:

* the whole step (dnum = 5 and the dnum = 1 variant) -- QKV (MHP) -> Q K^T -> masks, Softmax x V -> collapse -> W_O -> mask,
  FFN1 -> mask, FFN2 -> mask -- is bit-exact against the oracle's layer step
  (oracle/layer.py) on every masked ciphertext and every server share, including the
  per-inference mask ids (reading C19);
* the pipelined host-to-host run returns exactly the results of a plain step on
  device-resident inputs, for several steps in flight;
* consecutive inferences draw fresh masks (no reuse, Alg. 1 line 1 P:629)."""
import numpy as np
import pytest
import torch

import blb_inputs as bi
import oracle as O
import oracle.layer as OL

pytestmark = pytest.mark.gpu

blb = pytest.importorskip("paper_2508_19525_b200")
from paper_2508_19525_b200 import packing  # noqa: E402
from paper_2508_19525_b200.layer import Dims, FusedLinearLayer, LayerPipeline  # noqa: E402

L, D, H, FFN = 32, 64, 4, 128
BSGS = {"qkv": 8, "oproj": 4, "ffn1": 8, "ffn2": 4, "qk": 0}


def flat(res):
    out = []
    for _, _, r in res:
        out.extend(r if isinstance(r, (tuple, list)) else (r,))
    return out


@pytest.fixture(scope="module", params=["qktoy", "qktoy_dnum1"])
def setup(request):
    P = {"qktoy": bi.QKTOY, "qktoy_dnum1": bi.QKTOY_DNUM1}[request.param]
    params = blb.Params.from_preset(P)
    layer = FusedLinearLayer(params, Dims(L, D, H, FFN), bsgs=BSGS)
    rng = np.random.default_rng(7)
    W = [rng.normal(0.0, 0.04, s) for s in ((D, D), (D, D), (D, D), (D, D), (D, FFN), (FFN, D))]
    keys_key, enc_key, mask_key = bi.crypto_key(4, 77), bi.crypto_key(5, 77), bi.crypto_key(3, 77)
    keys, sk = blb.keygen(params, keys_key, layer.rotation_steps(), relin=True)
    layer.load_weights(*W)
    S = bi.softmax_rows(rng.normal(0.0, 1.0, (H, L, L)))
    V = rng.normal(0.0, 1.0, (H, L, D // H))
    sv_s, sv_v = packing.softmax_v_operands(S, V, params.n)
    slots = {"qkv": packing.spatial_slots(rng.normal(0, 1, (L, D)), params.n), "sv_s": sv_s, "sv_v": sv_v,
             "ffn1": packing.spatial_slots(rng.normal(0, 1, (L, D)), params.n),
             "ffn2": packing.spatial_slots(rng.normal(0, 1, (L, FFN)), params.n)}
    delta = 2.0 ** P.log_delta
    inputs, cid = {}, 0
    for name, zs in slots.items():
        pts = params.encode(torch.tensor(zs), delta, layer.level)
        inputs[name] = []
        for b in range(zs.shape[0]):
            inputs[name].append(blb.encrypt(params, sk, pts[b], layer.level, enc_key, 100 + cid, delta))
            cid += 1
    return dict(params=params, layer=layer, W=W, keys=keys, inputs=inputs, mask_key=mask_key, keys_key=keys_key,
                slots=slots, preset=P)


def test_layer_step_matches_oracle(setup):
    """dnum = 5 (alpha = 1, the fused ModUp / ModDown paths) and the dnum = 1 variant (one digit of
    all five ciphertext primes, four special primes: the generic base-conversion paths, C23)."""
    P = setup["preset"]
    pr = O.prime_chain(P.log_n, list(P.q_bits) + list(P.p_bits))
    ctx = O.Ctx(P.log_n, pr[:5], pr[5:], P.dnum)
    layer = setup["layer"]
    spec = OL.build(ctx, OL.LayerSpec(L, D, H, FFN, BSGS, layer.level), *setup["W"])
    assert OL.rotation_steps(spec) == layer.rotation_steps()
    okeys = O.keygen(ctx, setup["keys_key"], OL.rotation_steps(spec), relin=True)
    # the same ciphertexts on both sides (encryption is bit-exact, test_gpu_parity)
    oin = {k: [O.Ct(blb.to_numpy_u64(c.data), c.level, c.scale) for c in v] for k, v in setup["inputs"].items()}
    seq = 3
    ref = OL.layer_step(ctx, okeys, spec, oin, setup["mask_key"], seq)
    got = layer.step(setup["keys"], setup["inputs"], setup["mask_key"], seq=seq)
    names = sorted(name for name, _, _ in got)
    assert names == sorted(ref)
    for name, id0, (masked, share) in got:
        exp = ref[name]
        assert id0 == exp[0][0] and len(exp) == masked.shape[0]
        for t, (oid, om, osh) in enumerate(exp):
            assert oid == id0 + t
            assert np.array_equal(blb.to_numpy_u64(masked[t]), om), (name, t)
            assert np.array_equal(blb.to_numpy_u64(share[t]), osh), (name, t)


def test_masks_fresh_per_inference(setup):
    layer = setup["layer"]
    a = flat(layer.step(setup["keys"], setup["inputs"], setup["mask_key"], seq=10))
    b = flat(layer.step(setup["keys"], setup["inputs"], setup["mask_key"], seq=11))
    assert len(a) == len(b)
    for x, y in zip(a, b):
        assert not torch.equal(x, y)
    # the layer's own counter advances: two default calls never reuse a mask
    c = flat(layer.step(setup["keys"], setup["inputs"], setup["mask_key"]))
    d = flat(layer.step(setup["keys"], setup["inputs"], setup["mask_key"]))
    assert not any(torch.equal(x, y) for x, y in zip(c, d))


def test_layer_pipeline_matches_step(setup):
    layer, keys, mask_key, inputs = setup["layer"], setup["keys"], setup["mask_key"], setup["inputs"]
    refs = {s: [t.cpu() for t in flat(layer.step(keys, inputs, mask_key, seq=s))] for s in (21, 22)}
    assert all(t.numel() for t in refs[21])
    host_in = {k: [c.data.cpu().pin_memory() for c in v] for k, v in inputs.items()}
    pipe = LayerPipeline(layer, keys, mask_key, inputs)
    outs = [pipe.submit(host_in, seq=s) for s in (20, 21, 22)]  # three steps in flight, two buffer sets
    pipe.drain()
    torch.cuda.synchronize()
    # set 0 was reused by step 22, so compare step 21 (set 1) and step 22 (set 0)
    for got, s in ((outs[1], 21), (outs[2], 22)):
        assert len(got) == len(refs[s])
        for a, b in zip(got, refs[s]):
            assert torch.equal(a, b)
