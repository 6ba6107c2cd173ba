"""Weight-encode throughput (row a0) of the BERT-base layer plans on one GPU: seconds per plan
encode (blb_matmul_encode_weights: slot build, double-double FFT encode, NTT, blocked packing).

    python tools/bench_encode.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import blb_inputs as bi  # noqa: E402
import paper_2508_19525_b200 as blb  # noqa: E402
from paper_2508_19525_b200.layer import Dims, FusedLinearLayer  # noqa: E402

params = blb.Params.from_preset(bi.BERT)
layer = FusedLinearLayer(params, Dims(), bsgs=bi.BENCH_BSGS)
A = bi.bert_attention_inputs()
F = bi.bert_ffn_inputs()
res = {}
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    layer.load_weights(A["WQ"], A["WK"], A["WV"], F["WO"], F["W1"], F["W2"])
    torch.cuda.synchronize()
    res["load_weights_s_%d" % rep] = time.perf_counter() - t0
Wqkv = np.concatenate([A["WQ"], A["WK"], A["WV"]], axis=1)
for name, W in (("qkv", Wqkv), ("ffn1", F["W1"]), ("ffn2", F["W2"])):
    pl = layer.plans[name]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pl.encode_weights(W)
    torch.cuda.synchronize()
    res[name] = {"s": time.perf_counter() - t0, "plaintexts": pl.n_pt}
print(json.dumps(res))
