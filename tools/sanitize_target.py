"""compute-sanitizer target (tools/gpu.sh sanitize): the toy smoke (generic-N NTT, the bulk-copy
rings of k_mac_tma4 / k_mac_j, mask, ct-ct Q K^T) plus, at the BERT preset N = 2^16, one rotation,
a rescale, a small ct-pt MatMul and the mask -- the fused N = 2^16 NTT kernels (ModUp prologue,
ModDown epilogue), the key-switch inner product and the weight MAC ring at full size."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402
import blb_inputs as bi  # noqa: E402
import paper_2508_19525_b200 as blb  # noqa: E402

ge.smoke()
p = blb.Params.from_preset(bi.BERT)
plan = blb.MatmulPlan(p, 128, 256, 512, bsgs_B=4, level=4)
keys, sk = blb.keygen(p, bi.crypto_key(4, 9), plan.rotation_steps() + [1], relin=True)
z = np.random.default_rng(9).uniform(-1, 1, p.n)
ct = blb.encrypt(p, sk, p.encode(torch.tensor(z), 2.0 ** 40, 4), 4, bi.crypto_key(5, 9), 1, 2.0 ** 40)
r = blb.rotate(p, keys, ct, 1)
rs = blb.rescale(p, r)
W = np.random.default_rng(10).normal(0, 0.05, (256, 512))
out = plan(keys, [ct], plan.encode_weights(W))
m, s = blb.ckks_to_mpc(p, out, bi.crypto_key(3, 9), 5)
torch.cuda.synchronize()
print("sanitize target ok", rs.level, len(out), m.shape)
