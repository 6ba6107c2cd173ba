"""Row f4 throughput variant: the BERT-base ct-pt MatMuls (QKV, FFN1, FFN2 of the benched layer) on
`--batch` independent input sets -- sequential blb_ct_pt_matmul calls vs one blb_ct_pt_matmul_batch
(weight-stationary MAC: each plaintext tile read from HBM feeds two input sets).  Device time per input
set (CUDA events), after warm-up; prints one JSON line.

    python tools/bench_wsmac.py [--batch 2] [--steps 3] [--warmup 1]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import blb_inputs as bi  # noqa: E402
import paper_2508_19525_b200 as blb  # noqa: E402
from paper_2508_19525_b200 import packing  # noqa: E402
from paper_2508_19525_b200.layer import Dims, FusedLinearLayer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=2)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    dims = dict(bi.BERT_BASE)
    params = blb.Params.from_preset(bi.BERT, device=0)
    layer = FusedLinearLayer(params, Dims(**dims), 0, 1, bsgs=dict(bi.BENCH_BSGS))
    A = bi.bert_attention_inputs(dims["L"], dims["d"])
    F = bi.bert_ffn_inputs(dims["L"], dims["d"], dims["H"], dims["ffn"])
    keys, sk = blb.keygen(params, A["keys_key"], layer.rotation_steps(), relin=True)
    layer.load_weights(A["WQ"], A["WK"], A["WV"], F["WO"], F["W1"], F["W2"])
    shapes = {"qkv": (dims["L"], dims["d"]), "ffn1": (dims["L"], dims["d"]), "ffn2": (dims["L"], dims["ffn"])}
    sets = {}
    for name, (L, din) in shapes.items():
        sets[name] = []
        for b in range(args.batch):
            X = np.clip(np.random.default_rng(300 + b).normal(0, 1, (L, din)), -4, 4)
            z = packing.spatial_slots(X, params.n)
            sets[name].append([blb.encrypt(params, sk, params.encode(torch.tensor(z[t]), 2.0 ** 40, layer.level),
                                           layer.level, A["enc_key"], 5000 + 100 * b + t, 2.0 ** 40)
                               for t in range(z.shape[0])])
    del sk
    wss = {name: torch.empty(args.batch * layer.plans[name].workspace_bytes(layer.plans[name].n_out) // 8 + 1,
                             dtype=torch.int64, device="cuda") for name in shapes}

    def single():
        for name in shapes:
            pl = layer.plans[name]
            for b in range(args.batch):
                pl(keys, sets[name][b], layer.pts[name], ws=wss[name])

    def batched():
        for name in shapes:
            layer.plans[name].batch(keys, sets[name], layer.pts[name], ws=wss[name])

    out = {"workload": "BERT-base QKV + FFN1 + FFN2 ct-pt MatMuls (benched plans, N=2^16), %d input sets" % args.batch}
    for label, fn in (("sequential", single), ("weight_stationary", batched)):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out[label + "_ms_per_input"] = e0.elapsed_time(e1) / args.steps / args.batch
    print(json.dumps(out))


if __name__ == "__main__":
    main()
