"""Config 5 (GPT2-base, 12 layers): model.GPT2Stack keeps every layer's weights on the device (as compact
encode coefficients expanded before each MatMul, as float64 weights re-encoded per layer, or as resident
plaintexts).  The device encode equals the host-weight encode bit for bit, the compact coefficients
expand to exactly the encoded plaintexts, and a 2-layer stack returns, layer by layer and in every mode,
exactly what a freshly built layer with that layer's weights returns (itself pinned against the oracle
layer step in test_gpu_layer)."""
import numpy as np
import pytest
import torch

import blb_inputs as bi

pytestmark = pytest.mark.gpu

blb = pytest.importorskip("paper_2508_19525_b200")
from paper_2508_19525_b200 import packing  # noqa: E402
from paper_2508_19525_b200.layer import Dims, FusedLinearLayer  # noqa: E402
from paper_2508_19525_b200.model import GPT2Stack, gpt2_layer_weights  # noqa: E402

DIMS = Dims(32, 64, 4, 128)
BSGS = {"qkv": 8, "oproj": 4, "ffn1": 8, "ffn2": 4, "qk": 0}


def test_device_weight_encode_equals_host():
    params = blb.Params.from_preset(bi.QKTOY)
    W = np.random.default_rng(3).normal(0, 0.05, (64, 96))
    pl = blb.MatmulPlan(params, 32, 64, 96, bsgs_B=8, level=4)
    a = pl.encode_weights(W)
    b = pl.encode_weights(torch.tensor(W, dtype=torch.float64, device="cuda"))
    c = pl.encode_weights(torch.tensor(W, dtype=torch.float64, device="cuda"), out=torch.zeros_like(a))
    assert torch.equal(a, b) and torch.equal(a, c)


def inputs_for(params, layer, sk, seed):
    rng = np.random.default_rng(seed)
    S = bi.softmax_rows(rng.normal(0.0, 1.0, (DIMS.H, DIMS.L, DIMS.L)))
    V = rng.normal(0.0, 1.0, (DIMS.H, DIMS.L, DIMS.d // DIMS.H))
    sv_s, sv_v = packing.softmax_v_operands(S, V, params.n)
    slots = {"qkv": packing.spatial_slots(rng.normal(0, 1, (DIMS.L, DIMS.d)), params.n), "sv_s": sv_s, "sv_v": sv_v,
             "ffn1": packing.spatial_slots(rng.normal(0, 1, (DIMS.L, DIMS.d)), params.n),
             "ffn2": packing.spatial_slots(rng.normal(0, 1, (DIMS.L, DIMS.ffn)), params.n)}
    out, cid = {}, seed * 100
    for name, zs in slots.items():
        pts = params.encode(torch.tensor(zs), 2.0 ** 40, layer.level)
        out[name] = [blb.encrypt(params, sk, pts[b], layer.level, bi.crypto_key(5, 81), cid + b, 2.0 ** 40)
                     for b in range(zs.shape[0])]
        cid += zs.shape[0]
    return out


def test_compact_coeffs_expand_to_encode_weights():
    """blb_matmul_coeffs_to_pts(blb_matmul_encode_coeffs(W)) is bit-identical to blb_matmul_encode_weights(W),
    for a whole plan and for an output slice, at the toy ring and at N = 2^16."""
    for preset, (L, din, dout, B, lvl) in ((bi.QKTOY, (32, 64, 96, 8, 4)), (bi.BERT, (128, 256, 128, 4, 4))):
        params = blb.Params.from_preset(preset)
        W = np.random.default_rng(4).normal(0, 0.05, (din, dout))
        pl = blb.MatmulPlan(params, L, din, dout, bsgs_B=B, level=lvl)
        slices = [(0, pl.n_out)] + ([(1, pl.n_out - 2)] if pl.n_out >= 3 else [])
        for first, count in slices:
            ref = pl.encode_weights(W, first, count)
            coef = pl.encode_coeffs(torch.tensor(W, dtype=torch.float64, device="cuda"), first, count)
            got = pl.coeffs_to_pts(coef, first, count, out=torch.zeros_like(ref))
            torch.cuda.synchronize()
            assert torch.equal(got, ref)


def test_compact_coeffs_overflow_is_an_error():
    """Coefficients that need more than 40 bits are refused (BLB_E_OVERFLOW), never truncated."""
    params = blb.Params.from_preset(bi.QKTOY)
    pl = blb.MatmulPlan(params, 32, 64, 96, bsgs_B=8, level=4)
    W = np.random.default_rng(5).normal(0, 300.0, (64, 96))   # |scale * w| far above 2^39
    with pytest.raises(blb.BLBError):
        pl.encode_coeffs(W)


@pytest.mark.parametrize("mode", ["reencode", "resident", "coeffs"])
def test_two_layer_stack_matches_per_layer(mode):
    params = blb.Params.from_preset(bi.QKTOY)
    stack = GPT2Stack(params, 2, DIMS, bsgs=BSGS, mode=mode)
    assert stack.mode == mode
    keys, sk = blb.keygen(params, bi.crypto_key(4, 81), stack.rotation_steps(), relin=True)
    ins = [inputs_for(params, stack.layer, sk, 1 + l) for l in range(2)]
    mk = bi.crypto_key(3, 81)
    got = stack.step(keys, ins, mk, seq0=40)
    got2 = stack.step(keys, ins, mk, seq0=40)     # the second step re-encodes layer 0 again
    for l in range(2):
        ref_layer = FusedLinearLayer(params, DIMS, bsgs=BSGS)
        ref_layer.load_weights(*gpt2_layer_weights(l, DIMS))
        ref = ref_layer.step(keys, ins[l], mk, seq=40 + l)
        for g in (got, got2):
            assert [n for n, _, _ in g[l]] == [n for n, _, _ in ref]
            for (_, i0, (m0, s0)), (_, i1, (m1, s1)) in zip(g[l], ref):
                assert i0 == i1 and torch.equal(m0, m1) and torch.equal(s0, s1)
