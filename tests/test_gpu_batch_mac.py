"""Row f4: blb_ct_pt_matmul_batch (weight-stationary MAC over several input sets) returns, for every
set, exactly what blb_ct_pt_matmul returns for that set alone -- odd and even batch sizes (a pair of
sets per CTA, the last one alone), whole plan and an output slice, toy ring and N = 2^16."""
import numpy as np
import pytest
import torch

import blb_inputs as bi

pytestmark = pytest.mark.gpu

blb = pytest.importorskip("paper_2508_19525_b200")
from paper_2508_19525_b200 import packing  # noqa: E402


@pytest.mark.parametrize("preset,shape,nb", [(bi.QKTOY, (32, 64, 96, 8, 4), 3), (bi.BERT, (128, 256, 128, 4, 4), 2)])
def test_batch_equals_single(preset, shape, nb):
    L, din, dout, B, lvl = shape
    params = blb.Params.from_preset(preset)
    W = np.random.default_rng(7).normal(0, 0.05, (din, dout))
    pl = blb.MatmulPlan(params, L, din, dout, bsgs_B=B, level=lvl)
    keys, sk = blb.keygen(params, bi.crypto_key(4, 77), pl.rotation_steps())
    sets = []
    for b in range(nb):
        X = np.random.default_rng(100 + b).normal(0, 1, (L, din))
        z = packing.spatial_slots(X, params.n)
        sets.append([blb.encrypt(params, sk, params.encode(torch.tensor(z[t]), 2.0 ** 40, lvl), lvl,
                                 bi.crypto_key(5, 77), 1000 * b + t, 2.0 ** 40) for t in range(z.shape[0])])
    for first, count in [(0, pl.n_out)] + ([(1, pl.n_out - 1)] if pl.n_out >= 2 else []):
        pts = pl.encode_weights(W, first, count)
        got = pl.batch(keys, sets, pts, first, count)
        for b in range(nb):
            ref = pl(keys, sets[b], pts, first, count)
            for g, r in zip(got[b], ref):
                assert g.level == r.level and g.scale == r.scale and torch.equal(g.data, r.data), (b, first)
