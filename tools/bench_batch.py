"""Row f4 (throughput variant): batched same-user inputs packed along the spatial dimension
(App. D, "Batching enables BLB to pack more data along the spatial dimension, reduce
rotations").  B inputs of L = 128 tokens share one spatial block of L' = B L rows, so a ciphertext
holds c' = N / (2 L') columns; the ct-pt MatMuls (QKV with the MHP map, FFN1, FFN2) run unchanged on
plans built for L'.  Prints, per batch size, the device ms of the three MatMuls per call and per
input, their rotation counts, and plaintext bytes streamed (synthetic residues: encode is row a0).

    python tools/bench_batch.py [--batches 1,2,4] [--iters 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import blb_inputs as bi  # noqa: E402
import paper_2508_19525_b200 as blb  # noqa: E402


def plans_for(g, L, d=768, H=12, ffn=3072):
    c = g.n // L
    Bq = min(64, c)
    cm = blb.mhp_column_map(d, H, L, g.log_n)
    qkv_map = cm + [d + x if x >= 0 else -1 for x in cm] + list(range(2 * d, 3 * d))
    return {"qkv": blb.MatmulPlan(g, L, d, 3 * d, col_map=qkv_map, bsgs_B=Bq, level=4),
            "ffn1": blb.MatmulPlan(g, L, d, ffn, bsgs_B=Bq, level=4),
            "ffn2": blb.MatmulPlan(g, L, ffn, d, bsgs_B=min(16, c), level=4)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="1,2,4")
    ap.add_argument("--iters", type=int, default=3)
    args = ap.parse_args()
    g = blb.Params.from_preset(bi.BERT)
    k = 5
    res = []
    for B in [int(x) for x in args.batches.split(",")]:
        L = 128 * B
        plans = plans_for(g, L)
        steps = sorted({s for p in plans.values() for s in p.rotation_steps()})
        keys, _ = blb.keygen(g, bi.crypto_key(1, 1), steps, want_secret=False)
        ms = 0.0
        per = {}
        for name, p in plans.items():  # one MatMul's plaintexts resident at a time (16 L' k B per weight)
            pts = torch.randint(0, 2 ** 39, (p.n_pt, k, g.N), dtype=torch.int64, device="cuda")
            cts = [blb.Ciphertext(torch.randint(0, 2 ** 39, (2, k, g.N), dtype=torch.int64, device="cuda"), 4,
                                  2.0 ** 40) for _ in range(p.n_in)]
            ws = p.workspace()
            outs = p(keys, cts, pts, ws=ws)
            torch.cuda.synchronize()
            st = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(args.iters):
                p(keys, cts, pts, ws=ws, outs=outs)
            e1.record(st)
            torch.cuda.synchronize()
            per[name] = e0.elapsed_time(e1) / args.iters
            ms += per[name]
            del pts, cts, ws, outs
            torch.cuda.empty_cache()
        res.append({"batch": B, "L_spatial": L, "ms_per_call": ms, "ms_per_input": ms / B, "ms_per_matmul": per,
                    "rotations_per_input": sum(p.n_rotations for p in plans.values()) / B,
                    "plaintext_GB_per_input": sum(p.n_pt for p in plans.values()) * k * g.N * 8 / 1e9 / B})
        del keys
        torch.cuda.empty_cache()
    print(json.dumps({"workload": "BERT-base QKV(MHP) + FFN1 + FFN2 ct-pt MatMuls, N=2^16, batch packed "
                                  "along the spatial dimension", "results": res}))


if __name__ == "__main__":
    main()
